#!/bin/bash
# ncu source-level capture of the compress kernel (one launch each) at r=10 and r=1000 on the largest boundary
mkdir -p gpurun_out
for r in 10 1000; do
  ncu --set full --import-source on --clock-control none -k regex:"compress_kernel" -s 2 -c 1 \
      -o gpurun_out/src_r$r -f python scripts/profile_case.py --shape 64,256,56,56 --ratio $r --iters 3 > gpurun_out/src_r$r.log 2>&1
done
ls -la gpurun_out/src_r*.ncu-rep
