#!/bin/bash
# ncu source-level capture of one 24-CTA compress launch per (variant, ratio) on the largest boundary
#   RATIOS="10 100" bash scripts/gpu_prof_variant.sh base wu
mkdir -p gpurun_out
for v in "$@"; do
  for r in ${RATIOS:-10 100}; do
    GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so ncu --set full --import-source on --clock-control none -k regex:"compress_kernel" -s 2 -c 1 \
      -o gpurun_out/pv_${v}_r$r -f python scripts/profile_case.py --shape 64,256,56,56 --ratio $r --iters 3 --ctas 24 > gpurun_out/pv_${v}_r$r.log 2>&1
  done
done
ls -la gpurun_out/pv_*.ncu-rep
