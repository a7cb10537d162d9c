#!/bin/bash
# N=2 pull transport (trusted decompress) with library variants
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2410_12707_b200/_lib/variants/$v/libadatopk.so
  [ "$v" = "new" ] && lib=paper_2410_12707_b200/_lib/libadatopk.so
  GP_LIB=$lib GP_BENCH_DEC_MODE=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 \
    bench.py --gpus 2 --steps 10 --warmup 3 --no-pipeline --no-sweep --transport peer-pull > gpurun_out/pp2_$v.json 2> gpurun_out/pp2_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/pp2_$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', d['value'], d['ms_per_step'], r['frac'], r['launch_us_mean'], r.get('decompress_achieved'))" 2>/dev/null || (echo "$v ERR"; tail -5 gpurun_out/pp2_$v.err)
done
