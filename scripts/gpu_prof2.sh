cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/profile_case.py > gpurun_out/plain.log 2>&1 && python scripts/profile_case.py --shape 64,256,56,56 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^compress_kernel" -s 3 -c 1 -o gpurun_out/prof_c1b python scripts/profile_case.py > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^compress_kernel" -s 3 -c 1 -o gpurun_out/prof_r51 python scripts/profile_case.py --shape 64,256,56,56 > gpurun_out/ncu2.log 2>&1; echo ncu=$?
