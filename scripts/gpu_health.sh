mkdir -p gpurun_out/h
nvidia-smi -L > gpurun_out/h/gpus.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/h/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/h/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/h/smoke.log
timeout 600 python bench.py > gpurun_out/h/bench.json 2> gpurun_out/h/bench.err; echo "bench rc=$?" >> gpurun_out/h/bench.err
