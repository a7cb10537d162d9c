#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -x -q -p no:cacheprovider 2>&1 | tail -1
bash scripts/gpu_gt_ab.sh v2 new 2>&1 | grep -E "==|compress|cold"
for s in 4 8; do GP_E2E_STREAMS=$s timeout 600 python bench.py --steps 5 --warmup 3 --no-pipeline --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e streams', $s, d['e2e'])"; done
bash scripts/gpu_ab_r2.sh v2 new
