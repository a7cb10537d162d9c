cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/profile_case.py --shape 64,2048,7,7 --ratio 1000 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^compress_kernel" -s 3 -c 1 -o gpurun_out/prof_small python scripts/profile_case.py --shape 64,2048,7,7 --ratio 1000 > gpurun_out/ncu_small.log 2>&1; echo ncu=$?
