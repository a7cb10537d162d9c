mkdir -p gpurun_out/fin4
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/fin4/tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/fin4/tests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin4/smoke.log
timeout 900 python bench.py > gpurun_out/fin4/bench.json 2> gpurun_out/fin4/bench.err; echo "rc=$?" >> gpurun_out/fin4/bench.err
