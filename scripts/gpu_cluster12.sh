mkdir -p gpurun_out/cl12
timeout 300 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/cl12/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/cl12/tests_cluster.log
for rule in 0 1; do
  GP_CL_NC_RULE=$rule timeout 300 python scripts/cluster_probe.py --small --out gpurun_out/cl12/small_rule$rule.json > gpurun_out/cl12/small_rule$rule.log 2>&1
done
