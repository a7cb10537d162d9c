#!/bin/bash
# A/B of library variants on one ratio class of the bench workload at a time (GP_BENCH_ONLY_R)
#   bash scripts/gpu_ab_ratio.sh cur wu
mkdir -p gpurun_out
for r in 10 100 1000; do
  for v in "$@"; do
    GP_BENCH_ONLY_R=$r GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep \
      > gpurun_out/abr_${v}_$r.json 2> gpurun_out/abr_${v}_$r.err
    python -c "import json; d=json.loads(open('gpurun_out/abr_${v}_$r.json').read().strip().splitlines()[-1]); print('r=$r', '$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us_mean'])" 2>/dev/null || echo "r=$r $v ERR"
  done
done
