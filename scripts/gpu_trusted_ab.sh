#!/bin/bash
for rep in 1 2; do
  for m in 0 2; do
    GP_BENCH_DEC_MODE=$m timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dec_mode', $m, 'rep', $rep, d['value'], d['roofline']['frac'], round(d['roofline']['decompress_achieved']))"
  done
done
