#!/bin/bash
# per-phase compress timing (scripts/graph_timing.py) for library variants: bash scripts/gpu_gt_ab.sh v1 new
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "new" ]; then lib=paper_2410_12707_b200/_lib/libadatopk.so; else lib=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so; fi
  echo "== $v"
  GP_LIB=$lib GT_SHAPES="C1,7x7,28x28" timeout 600 python scripts/graph_timing.py 10,100 2>&1 | grep -v Warning
done
