#!/bin/bash
# A/B of library variants at N=1: bench without the pipeline and sweep sub-measurements, two alternating repetitions
#   bash scripts/gpu_ab_fast.sh base v1 v2 ...   (paper_2410_12707_b200/_lib/variants/<name>)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep \
      > gpurun_out/abf_${v}_$rep.json 2> gpurun_out/abf_${v}_$rep.err
  done
done
