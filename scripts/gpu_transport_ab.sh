# N>1 bench, copy-engine peer copies vs fused peer stores, alternating (development aid); N from env (default 2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
N=${N:-2}
for r in 1 2; do
for t in peer peer-store; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + r)) \
  bench.py --gpus $N --no-pipeline --transport $t > gpurun_out/bench_n${N}_${t}_$r.json 2> gpurun_out/bench_n${N}_${t}_$r.err
echo $t$r=$? $(python -c "import json;j=json.loads(open('gpurun_out/bench_n${N}_${t}_$r.json').read().splitlines()[-1]);print(j['value'],j['ms_per_step'],j['e2e']['value'])" 2>&1 | tail -1)
done
done
