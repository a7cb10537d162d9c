#!/bin/bash
# N=2: graph-replayed vs eager timed steps
mkdir -p gpurun_out
for g in "" "--no-graph"; do
  tag=${g:-graph}
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 \
    bench.py --gpus 2 --steps 10 --warmup 3 --no-pipeline --no-sweep $g > gpurun_out/n2e_$tag.json 2> gpurun_out/n2e_$tag.err
  python -c "import json; d=json.loads(open('gpurun_out/n2e_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$tag', d['value'], d['ms_per_step'], r['frac'], r['launch_us_mean'])" 2>/dev/null || (echo "$tag ERR"; tail -3 gpurun_out/n2e_$tag.err)
done
