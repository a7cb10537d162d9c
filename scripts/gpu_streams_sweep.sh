#!/bin/bash
# bench value vs the number of concurrent streams (compress grid = 148 / streams), two alternating passes
for rep in 1 2; do
  for s in 4 5 6 8; do
    timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-sweep --streams $s 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('streams', $s, 'rep', $rep, d['value'], d['roofline']['frac'], round(d['roofline']['decompress_achieved']))"
  done
done
