"""One small workload for ncu: compress + decompress of the C1 tensor (8x1024x768 fp32, r=100).

    python scripts/profile_case.py [--shape 8,1024,768] [--ratio 100] [--iters 5]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="8,1024,768")
    ap.add_argument("--ratio", type=float, default=100.0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--ctas", type=int, default=0, help="compress grid cap (0: one CTA per SM)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    shape = tuple(int(s) for s in args.shape.split(","))
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(shape, device=dev, generator=g).reshape(-1)
    code = 0
    if args.dtype == "bf16":
        x = x.to(torch.bfloat16)
        code = 1
    L = _lib.lib()
    d = x.numel()
    k = P.select_k(d, args.ratio)
    st = torch.cuda.current_stream().cuda_stream
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
    wsb = L.gp_topk_workspace_bytes(d, code)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    assert L.gp_workspace_init(ws.data_ptr(), wsb, st) == 0
    out = torch.empty(d, dtype=x.dtype, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    for _ in range(args.iters):
        flush.sum()
        assert L.gp_topk_compress_frame_ctas(x.data_ptr(), code, d, k, frame.data_ptr(), ws.data_ptr(), wsb, st,
                                             args.ctas) == 0
        assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), code, 0, err.data_ptr(), st) == 0
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    print(f"ok d={d} k={k}")


if __name__ == "__main__":
    main()
