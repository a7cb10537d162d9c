"""GPT-2 compressed-pipeline throughput (BASELINE.json configs[2] and configs[3]).

    python scripts/pipeline_bench.py --model medium                      # 1 GPU, no boundary
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/pipeline_bench.py --model medium --plan uniform
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/pipeline_bench.py --model xl --plan adatopk

Prints one JSON line (rank 0).  Synthetic tokens, random-init weights.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2410_12707_b200 import pipeline as PL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="medium", choices=sorted(PL.MODELS))
    ap.add_argument("--micro-batch", type=int, default=None)
    ap.add_argument("--n-micro", type=int, default=None)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--plan", default="uniform", choices=["none", "uniform", "adatopk", "measured"])
    ap.add_argument("--ratio", type=float, default=100.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    line = PL.run_pipeline(args.model, args.plan, args.ratio, args.micro_batch, args.n_micro, args.seq, args.steps,
                           args.warmup)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
