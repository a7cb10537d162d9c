#!/bin/bash
# ncu source-level capture of the compress kernel (one launch each) on the largest boundary, bench-sized 24-CTA grid
mkdir -p gpurun_out
for r in ${RATIOS:-10 100}; do
  ncu --set full --import-source on --clock-control none -k regex:"compress_kernel" -s 2 -c 1 \
      -o gpurun_out/src24_r$r -f python scripts/profile_case.py --shape 64,256,56,56 --ratio $r --iters 3 --ctas 24 > gpurun_out/src24_r$r.log 2>&1
done
ls -la gpurun_out/src24_r*.ncu-rep
