#!/bin/bash
# N=2 bench with 1..7 copy streams for the frame pushes
mkdir -p gpurun_out
for cs in "$@"; do
  GP_BENCH_COPY_STREAMS=$cs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
    bench.py --gpus 2 --steps 10 --warmup 3 --no-pipeline --no-sweep > gpurun_out/n2cs_$cs.json 2> gpurun_out/n2cs_$cs.err
  python -c "import json; d=json.loads(open('gpurun_out/n2cs_$cs.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cs=$cs', d['value'], d['ms_per_step'], r['frac'], r['launch_us_mean'], d['transfer']['peer_copy_gbs'])" 2>/dev/null || (echo "cs=$cs ERR"; tail -3 gpurun_out/n2cs_$cs.err)
done
