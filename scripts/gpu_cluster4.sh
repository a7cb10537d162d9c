mkdir -p gpurun_out/cl4
timeout 300 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/cl4/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/cl4/tests_cluster.log
timeout 300 python scripts/cluster_probe.py --small --out gpurun_out/cl4/small.json > gpurun_out/cl4/small.log 2>&1
timeout 300 python scripts/cluster_probe.py --out gpurun_out/cl4/large.json > gpurun_out/cl4/large.log 2>&1
timeout 300 python scripts/cluster_stamps.py > gpurun_out/cl4/stamps.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/cl4/tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/cl4/tests_all.log
