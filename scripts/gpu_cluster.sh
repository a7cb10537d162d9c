# single-cluster compress: parity tests, A/B probe, then the whole GPU suite
mkdir -p gpurun_out/cl
timeout 420 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/cl/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/cl/tests_cluster.log
if grep -q 'rc=0' gpurun_out/cl/tests_cluster.log; then
  timeout 600 python scripts/cluster_probe.py --out gpurun_out/cl/cluster_probe.json > gpurun_out/cl/probe.log 2>&1; echo "rc=$?" >> gpurun_out/cl/probe.log
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/cl/tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/cl/tests_all.log
fi
