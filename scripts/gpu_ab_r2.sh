#!/bin/bash
# A/B: bench (no pipeline) alternating library variants on one box.
#   bash scripts/gpu_ab_r2.sh base new ...   (variant "new" = the in-tree library)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = "new" ]; then lib=paper_2410_12707_b200/_lib/libadatopk.so; else lib=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so; fi
    GP_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
  done
done
python scripts/ab_summary.py "$@"
