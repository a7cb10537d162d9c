#!/bin/bash
# N=2 transports with the trusted decompress (no sortedness re-read of the frame)
mkdir -p gpurun_out
b2() { tag=$1; shift; env GP_X=0 "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --gpus 2 --steps 10 --warmup 3 --no-pipeline --no-sweep $T > gpurun_out/pp_$tag.json 2> gpurun_out/pp_$tag.err; }
T="--transport peer-pull" b2 pull0 GP_BENCH_DEC_MODE=0
T="--transport peer-pull" b2 pull2 GP_BENCH_DEC_MODE=2
T="--transport peer" b2 push2 GP_BENCH_DEC_MODE=2
T="--transport peer" b2 push0 GP_BENCH_DEC_MODE=0
for t in pull0 pull2 push2 push0; do
  python -c "import json; d=json.loads(open('gpurun_out/pp_$t.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$t', d['value'], d['ms_per_step'], r['frac'], r['launch_us_mean'], r.get('decompress_achieved'))" 2>/dev/null || (echo "$t ERR"; tail -5 gpurun_out/pp_$t.err)
done
