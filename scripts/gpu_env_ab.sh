# N-rank bench (no pipeline), A/B over an environment setting, alternating twice (development aid)
#   N=2 A="GP_BENCH_STAGGER=1" B="GP_BENCH_STAGGER=0" bash scripts/gpu_env_ab.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
N=${N:-2}
for r in 1 2; do
for tag in A B; do
eval "envs=\$$tag"
env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + r)) \
  bench.py --gpus $N --no-pipeline $EXTRA > gpurun_out/envab_${tag}_$r.json 2> gpurun_out/envab_${tag}_$r.err
echo "$tag($envs)$r=$? $(python -c "import json;j=json.loads(open('gpurun_out/envab_${tag}_$r.json').read().splitlines()[-1]);print(j['value'],j['ms_per_step'])" 2>&1 | tail -1)"
done
done
