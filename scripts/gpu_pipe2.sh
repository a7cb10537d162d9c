cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
for b in 0 1; do for nm in 4 8; do
GP_P2P_BATCHED=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2956$nm scripts/pipeline_bench.py --model medium --plan uniform --ratio 100 --steps 3 --warmup 1 --n-micro $nm 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('batched=$b n_micro=$nm', j['value'], j['ms_per_step'])"
done; done
