cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpus.txt
timeout 300 python -m pytest tests/test_transport.py -m gpu -q -p no:cacheprovider > gpurun_out/multi_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/multi_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench2=$?
tail -3 gpurun_out/bench2.err
