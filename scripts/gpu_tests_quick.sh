#!/bin/bash
# GPU test suite + smoke + a short bench (one GPU)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
if [ "$1" = "bench" ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 --no-pipeline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
fi
tail -n 3 gpurun_out/smoke.log gpurun_out/gputests.log
