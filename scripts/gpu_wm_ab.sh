#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -x -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/gpu_gt_ab.sh wm0 new 2>&1 | grep -E "==|compress"
bash scripts/gpu_ab_r2.sh wm0 new
