#!/bin/bash
# A/B of the candidate-list L2 policy variants at N=1, with and without the N>1 copy pattern (local copies)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    lib=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so
    GP_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep > gpurun_out/l2_${v}_$rep.json 2> gpurun_out/l2_${v}_$rep.err
    GP_LIB=$lib GP_BENCH_LOCALCOPY=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep > gpurun_out/l2lc_${v}_$rep.json 2> gpurun_out/l2lc_${v}_$rep.err
  done
done
