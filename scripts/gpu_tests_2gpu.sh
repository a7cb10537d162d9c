mkdir -p gpurun_out/g2
nvidia-smi -L > gpurun_out/g2/gpus.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/g2/tests.log 2>&1; echo "rc=$?" >> gpurun_out/g2/tests.log
