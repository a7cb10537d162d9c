# final state: cluster parity, A/B probes, stamps, whole GPU suite, smoke, bench N=1
mkdir -p gpurun_out/fin3
timeout 300 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/fin3/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/fin3/tests_cluster.log
timeout 300 python scripts/cluster_probe.py --small --out gpurun_out/fin3/small.json > gpurun_out/fin3/small.log 2>&1
timeout 300 python scripts/cluster_probe.py --out gpurun_out/fin3/large.json > gpurun_out/fin3/large.log 2>&1
GP_CLUSTER_PATH=2 timeout 300 python scripts/cluster_stamps.py > gpurun_out/fin3/stamps.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/fin3/tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/fin3/tests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin3/smoke.log
timeout 900 python bench.py > gpurun_out/fin3/bench.json 2> gpurun_out/fin3/bench.err; echo "rc=$?" >> gpurun_out/fin3/bench.err
