mkdir -p gpurun_out/cl2
timeout 300 python scripts/cluster_stamps.py > gpurun_out/cl2/stamps.log 2>&1; echo "rc=$?" >> gpurun_out/cl2/stamps.log
timeout 600 python scripts/cluster_probe.py --out gpurun_out/cl2/cluster_probe.json > gpurun_out/cl2/probe.log 2>&1; echo "rc=$?" >> gpurun_out/cl2/probe.log
