mkdir -p gpurun_out/cl11
timeout 300 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/cl11/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/cl11/tests_cluster.log
if grep -q 'rc=0' gpurun_out/cl11/tests_cluster.log; then
timeout 300 python scripts/cluster_probe.py --small --out gpurun_out/cl11/small.json > gpurun_out/cl11/small.log 2>&1
timeout 300 python scripts/cluster_probe.py --out gpurun_out/cl11/large.json > gpurun_out/cl11/large.log 2>&1
GP_CLUSTER_PATH=2 timeout 300 python scripts/cluster_stamps.py > gpurun_out/cl11/stamps.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:compress_cluster -c 1 -s 2 -o gpurun_out/cl11/cluster python scripts/cluster_one.py > gpurun_out/cl11/ncu.log 2>&1
fi
