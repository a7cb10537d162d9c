cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench2=$?; tail -2 gpurun_out/bench2.err
