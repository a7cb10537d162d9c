#!/bin/bash
# Does the N>1 frame copy slow the compress phase through this GPU's own copies or the peer's incoming writes?
mkdir -p gpurun_out
b1() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-pipeline --no-sweep > gpurun_out/cp_$tag.json 2> gpurun_out/cp_$tag.err; }
b2() { tag=$1; shift; env GP_X=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 \
    bench.py --gpus 2 --steps 10 --warmup 3 --no-pipeline --no-sweep "$@" > gpurun_out/cp_$tag.json 2> gpurun_out/cp_$tag.err; }
b1 n1 GP_X=0
b1 n1lc GP_BENCH_LOCALCOPY=1
b1 n1lc_dec0 GP_BENCH_LOCALCOPY=1 GP_BENCH_DEC_MODE=0
b2 n2store --transport peer-store
b2 n2nccl --transport nccl
b1 n1lc2 GP_BENCH_LOCALCOPY=1
