#!/bin/bash
# ncu launch lists of one timed bench step in its timed configuration (4 streams, CUDA-graph replay,
# 24 distinct inputs): the 24 compress and 24 decompress kernel nodes of the first timed-region replay.
# eager launches before it: 1 + GP_BENCH_SPINUP(0) + warmup(3) steps + 1 pre-capture step = 5 x 24 per kernel.
mkdir -p gpurun_out
export GP_BENCH_SPINUP=0
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"^compress_kernel" -s 120 -c 24 --csv --log-file gpurun_out/launches_c.csv \
  python bench.py --no-pipeline --no-sweep --steps 1 --warmup 3 > gpurun_out/ncu_c.log 2>&1; echo "ncu c=$?"
ncu --metrics $M --clock-control none -k regex:"decompress" -s 120 -c 24 --csv --log-file gpurun_out/launches_d.csv \
  python bench.py --no-pipeline --no-sweep --steps 1 --warmup 3 > gpurun_out/ncu_d.log 2>&1; echo "ncu d=$?"
# one --set full capture of the dominant kernel: the largest r=10 compress inside the graph replay
ncu --set full --import-source on --clock-control none -k regex:"^compress_kernel" -s 120 -c 24 \
  -o gpurun_out/full_r02 -f python bench.py --no-pipeline --no-sweep --steps 1 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full=$?"
ls -la gpurun_out/launches_*.csv gpurun_out/full_r02.ncu-rep
