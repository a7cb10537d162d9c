mkdir -p gpurun_out/ncl
python scripts/cluster_one.py > gpurun_out/ncl/run.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:compress_cluster -c 1 -s 2 -o gpurun_out/ncl/cluster python scripts/cluster_one.py > gpurun_out/ncl/ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ncl/ncu.log
