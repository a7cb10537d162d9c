#!/bin/bash
# A/B of library variants across stream counts (bench without pipeline/sweep)
#   STREAMS="1 3 6" bash scripts/gpu_ab_streams.sh base wu
mkdir -p gpurun_out
for s in ${STREAMS:-1 3 6}; do
  for v in "$@"; do
    GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep --streams $s \
      > gpurun_out/abs_${v}_s$s.json 2> gpurun_out/abs_${v}_s$s.err
  done
done
for s in ${STREAMS:-1 3 6}; do for v in "$@"; do
  python -c "import json,sys; d=json.loads(open('gpurun_out/abs_${v}_s$s.json').read().strip().splitlines()[-1]); print('s$s', '$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us_mean'])" 2>/dev/null || echo "s$s $v ERR"
done; done
