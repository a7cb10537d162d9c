cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 120 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests.log
timeout 300 python scripts/quick_timing.py > gpurun_out/timing.log 2>&1; echo "timing rc=$?"
cat gpurun_out/timing.log | tail -20
