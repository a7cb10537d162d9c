cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/profile_case.py --shape 64,256,56,56 --ratio 10 --ctas 37 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^compress_kernel" -s 3 -c 1 -o gpurun_out/prof_dense python scripts/profile_case.py --shape 64,256,56,56 --ratio 10 --ctas 37 > gpurun_out/ncu_dense.log 2>&1; echo ncu=$?
