#!/bin/bash
# N=2 (and N=4 if present): per-frame hand-off vs one hand-off per step
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -le $N ] || continue
  for fh in 1 0; do
    GP_BENCH_FRAME_HANDOFF=$fh timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29523 \
      bench.py --gpus $n --steps 10 --warmup 3 --no-pipeline --no-sweep > gpurun_out/n${n}f_$fh.json 2> gpurun_out/n${n}f_$fh.err
    python -c "import json; d=json.loads(open('gpurun_out/n${n}f_$fh.json').read().strip().splitlines()[-1]); r=d['roofline']; print('n=$n fh=$fh', d['value'], d['ms_per_step'], r['frac'], r['launch_us_mean'])" 2>/dev/null || (echo "n=$n fh=$fh ERR"; tail -5 gpurun_out/n${n}f_$fh.err)
  done
done
