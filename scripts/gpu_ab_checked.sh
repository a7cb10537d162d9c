#!/bin/bash
# parity subset + A/B (v1 vs in-tree) + the checked variant through the sanitizer driver
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -x -q -p no:cacheprovider 2>&1 | tail -2
GP_LIB=paper_2410_12707_b200/_lib/variants/checked/libadatopk.so timeout 600 python scripts/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo "checked rc=$?" >> gpurun_out/checked_cases.log
tail -n 2 gpurun_out/checked_cases.log
bash scripts/gpu_ab_r2.sh "$@"
