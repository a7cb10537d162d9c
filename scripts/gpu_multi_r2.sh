#!/bin/bash
# multi-GPU round-2 run: 2-GPU tests, bench at N=1/2/4 (one box, 4 GPUs)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "world2 or dist_pipeline or measured or nccl or peer or another_device" > gpurun_out/multi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/multi_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
for n in 2 4; do
  [ $n -le $N ] || continue
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r2_bench$n.json 2> gpurun_out/r2_bench$n.err
done
tail -n 3 gpurun_out/multi_tests.log; for f in gpurun_out/r2_bench*.json; do echo $f; head -c 300 $f; echo; done
