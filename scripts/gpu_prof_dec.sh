cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/profile_case.py --shape ${SHAPE:-64,256,56,56} --ratio ${RATIO:-10} > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"decompress" -s 3 -c 1 -o gpurun_out/prof_dec python scripts/profile_case.py --shape ${SHAPE:-64,256,56,56} --ratio ${RATIO:-10} > gpurun_out/ncu_dec.log 2>&1; echo ncu=$?
