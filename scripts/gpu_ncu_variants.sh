#!/bin/bash
# per-unit compress launch list (time, instructions) of one timed bench step, per library variant
#   bash scripts/gpu_ncu_variants.sh base wu
mkdir -p gpurun_out
export GP_BENCH_SPINUP=0
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum
for v in "$@"; do
  GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so ncu --metrics $M --clock-control none -k regex:"^compress_kernel" -s 120 -c 24 --csv \
    --log-file gpurun_out/nv_$v.csv python bench.py --no-pipeline --no-sweep --steps 1 --warmup 3 > gpurun_out/nv_$v.log 2>&1; echo "$v rc=$?"
done
