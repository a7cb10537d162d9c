"""Per-warp stream timeline from WSTAMP cycle stamps (development aid).

    python scripts/warp_timeline.py [--shape 64,2048,7,7] [--ratio 1000]
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="64,2048,7,7")
    ap.add_argument("--ratio", type=float, default=1000)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    L.gp_debug_stamps.argtypes = [ctypes.c_void_p]
    shape = tuple(int(v) for v in args.shape.split(","))
    x = torch.randn(shape, device=dev).reshape(-1)
    d = x.numel()
    k = P.select_k(d, args.ratio)
    st = torch.cuda.current_stream().cuda_stream
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
    wsb = L.gp_topk_workspace_bytes(d, 0)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    L.gp_workspace_init(ws.data_ptr(), wsb, st)
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    dbg = torch.zeros(32768 + 1024 * 32 * 16, dtype=torch.int64, device=dev)
    for it in range(3):
        L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, st)
    flush.sum()
    torch.cuda.synchronize()
    L.gp_debug_stamps(dbg.data_ptr())
    L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, st)
    torch.cuda.synchronize()
    L.gp_debug_stamps(None)
    a = dbg.cpu().numpy()
    cta = a[:32768].reshape(1024, 32)
    G = int((cta[:, 0] > 0).sum())
    # cycles per ns from CTA stamps (globaltimer vs clock64)
    ns, cy = cta[:G, :9].astype(np.float64), cta[:G, 16:25].astype(np.float64)
    f = np.median((cy[:, 8] - cy[:, 0]) / np.maximum(ns[:, 8] - ns[:, 0], 1))
    w = a[32768:32768 + G * 32 * 16].reshape(G * 32, 16).astype(np.float64)
    base = w[:, 0:1]
    rel = (w - base) / f / 1e3  # us since the warp's start
    names = ["start", "row0 in"] + [f"row{r}" for r in range(12)] + ["loop end", "flushed"]
    print(f"d={d} k={k} G={G} clock {f:.3f} GHz; per-warp us since warp start (mean / p90 / max)")
    for i, nm in enumerate(names):
        col = rel[:, i][w[:, i] > 0]
        if col.size:
            print(f"  {nm:10s} n={col.size:5d}  {col.mean():7.2f} {np.percentile(col, 90):7.2f} {col.max():7.2f}")
    # CTA-level stage ends (globaltimer) for reference
    t0 = ns[:, 0].min()
    print("  CTA stamps (us from first CTA start):", " ".join(f"{np.mean(ns[:, i] - t0) / 1e3:.2f}" for i in range(9)))


if __name__ == "__main__":
    main()
