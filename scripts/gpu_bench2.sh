cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
N=${N:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus $N > gpurun_out/bench$N.json 2> gpurun_out/bench$N.err; echo bench$N=$?; tail -2 gpurun_out/bench$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus $N --impl reference > gpurun_out/bench${N}_ref.json 2> gpurun_out/bench${N}_ref.err; echo ref$N=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29553 scripts/pipeline_bench.py --model medium --plan uniform --ratio 100 --steps 3 --warmup 2 --n-micro 8 > gpurun_out/pipe$N.json 2> gpurun_out/pipe$N.err; echo pipe$N=$?
