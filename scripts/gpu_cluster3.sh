mkdir -p gpurun_out/cl3
for m in 1024 2048 4096 8192 65536; do
  GP_CL_MIN_PER_CTA=$m timeout 300 python scripts/cluster_probe.py --small --out gpurun_out/cl3/small_$m.json > gpurun_out/cl3/small_$m.log 2>&1
done
timeout 300 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/cl3/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/cl3/tests_cluster.log
