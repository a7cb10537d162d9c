"""A/B of the single-cluster compress (gp_cluster.cu) against the cooperative
grid on short vectors: compress and decompress device time per launch inside a
CUDA graph, each launch after a 512 MB L2 read flush (differenced against the
flush alone, as scripts/sweep.py does), and warm (no flush), plus the frame
equality of the two paths.

    python scripts/cluster_probe.py [--out gpurun_out/cluster_probe.json] [--small]

--small: vectors of 1K..64K elements (the default routing's threshold); the
CTA count per cluster follows GP_CL_MIN_PER_CTA (elements per CTA, env).
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402
from scripts.graph_timing import graph_time  # noqa: E402

CASES = [  # (dtype, d)
    ("fp32", 65_536), ("fp32", 131_072), ("fp32", 196_608), ("fp32", 262_144), ("fp32", 393_216),
    ("bf16", 262_144), ("bf16", 524_288), ("bf16", 786_432), ("fp64", 65_536), ("fp64", 131_072),
]
SMALL = [("fp32", 1024), ("fp32", 4096), ("fp32", 8192), ("fp32", 16_384), ("fp32", 32_768), ("fp32", 65_536),
         ("bf16", 16_384), ("bf16", 65_536), ("fp64", 8192), ("fp64", 32_768)]
RATIOS = [10, 100, 1000]
TORCH = {"fp32": torch.float32, "bf16": torch.bfloat16, "fp64": torch.float64}
CODE = {"fp32": 0, "bf16": 1, "fp64": 2}
ESZ = {"fp32": 4, "bf16": 2, "fp64": 8}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--small", action="store_true")
    args = ap.parse_args()
    cases, ratios = (SMALL, [10, 100]) if args.small else (CASES, RATIOS)
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    rows = []
    for dt, d in cases:
        code = CODE[dt]
        g = torch.Generator(device=dev).manual_seed(d)
        x = torch.randn(d, device=dev, generator=g).to(TORCH[dt])
        wsb = L.gp_topk_workspace_bytes(d, code)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        L.gp_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
        out = torch.empty(d, dtype=x.dtype, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        for r in ratios:
            k = P.select_k(d, r)
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)

            def fl():
                flush.sum()

            def comp():
                assert L.gp_topk_compress_frame(x.data_ptr(), code, d, k, frame.data_ptr(), ws.data_ptr(), wsb,
                                                torch.cuda.current_stream().cuda_stream) == 0

            def dec():
                assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), code, 0, err.data_ptr(),
                                                  torch.cuda.current_stream().cuda_stream) == 0

            row = {"dtype": dt, "d": d, "mb": round(d * ESZ[dt] / 2**20, 2), "ratio": r, "k": k}
            frames = {}
            for path in (2, 0):
                L.gp_set_cluster_path(path)
                t0 = graph_time([fl], n=10, reps=5)
                tc = graph_time([fl, comp], n=10, reps=5) - t0
                tp = graph_time([fl, comp, dec], n=10, reps=5) - t0
                warm = graph_time([comp], n=50, reps=5)
                warm_pair = graph_time([comp, dec], n=50, reps=5)
                torch.cuda.synchronize()
                comp()
                torch.cuda.synchronize()
                frames[path] = bytes(frame.cpu().numpy())
                tag = "cluster" if path else "coop"
                row[f"{tag}_compress_us"] = round(tc, 2)
                row[f"{tag}_pair_us"] = round(tp, 2)
                row[f"{tag}_warm_compress_us"] = round(warm, 2)
                row[f"{tag}_warm_pair_us"] = round(warm_pair, 2)
            L.gp_set_cluster_path(1)
            row["min_per_cta"] = os.environ.get("GP_CL_MIN_PER_CTA", "4096")
            row["frames_equal"] = frames[0] == frames[2]
            row["speedup_compress"] = round(row["coop_compress_us"] / row["cluster_compress_us"], 2)
            print(json.dumps(row), flush=True)
            rows.append(row)
    if args.out:
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps({"rows": rows}, indent=1))


if __name__ == "__main__":
    main()
