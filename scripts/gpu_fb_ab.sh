#!/bin/bash
for v in fb3 fb5; do
  GP_LIB=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
done
bash scripts/gpu_gt_ab.sh new fb3 fb5
bash scripts/gpu_ab_r2.sh new fb3 fb5
