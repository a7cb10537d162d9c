#!/bin/bash
# round-2 one-GPU measurement: GPU tests, smoke, bench N=1 + reference arm, sweep (with the CPU reference leg)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
if [ "$1" = "full" ]; then
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref1.json 2> gpurun_out/r2_ref1.err
  timeout 1800 python scripts/sweep.py --out gpurun_out/sweep_r02.json > gpurun_out/sweep_r02.log 2>&1
fi
tail -n 3 gpurun_out/smoke.log gpurun_out/gputests.log
