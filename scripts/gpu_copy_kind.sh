#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/copy_kind_probe.py > gpurun_out/copykind.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/copykind_ncu.csv python scripts/copy_kind_probe.py >> gpurun_out/copykind.log 2>&1
GP_BENCH_LOCALCOPY=1 GP_BENCH_SPINUP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 300 --log-file gpurun_out/lc_ncu.csv python bench.py --steps 1 --warmup 3 --no-pipeline --no-sweep >> gpurun_out/copykind.log 2>&1
