#!/bin/bash
# N=2 overhead probe: where do the extra ~0.27 ms per step at N>1 go?
mkdir -p gpurun_out
timeout 300 python scripts/pcie_probe.py > gpurun_out/pcie.log 2>&1
run() {  # tag, env..., -- args
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 2 --steps 10 --warmup 3 --no-pipeline --no-sweep > gpurun_out/n2_$tag.json 2> gpurun_out/n2_$tag.err
}
run base GP_X=0
run nocopy GP_BENCH_NOCOPY=1
run dec2 GP_BENCH_DEC_MODE=2
run cs2 GP_BENCH_COPY_STREAMS=2
run base2 GP_X=0
