#!/bin/bash
# bench (no pipeline/sweep) for one library variant under a list of env settings
#   bash scripts/gpu_env_sweep.sh VARIANT "A=1 B=2" "A=3" ...
mkdir -p gpurun_out
v=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  env $e GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep \
    > gpurun_out/es_${v}_$i.json 2> gpurun_out/es_${v}_$i.err
  python -c "import json; d=json.loads(open('gpurun_out/es_${v}_$i.json').read().strip().splitlines()[-1]); print('$v', '$e', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_us_mean'])" 2>/dev/null || echo "$v $e ERR"
done
