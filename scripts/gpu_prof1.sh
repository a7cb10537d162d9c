cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python scripts/quick_timing.py > gpurun_out/timing4.log 2>&1; echo rc=$?
GP_NO_PREFETCH=1 timeout 300 python scripts/quick_timing.py > gpurun_out/timing4_nopf.log 2>&1; echo rc=$?
python scripts/profile_case.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"compress_kernel|decompress_kernel" -s 6 -c 2 -o gpurun_out/prof_c1 python scripts/profile_case.py > gpurun_out/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu.log
