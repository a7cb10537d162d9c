"""Per-CTA stage stamps of one decompress launch (development aid)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402

L = _lib.lib()
L.gp_debug_dec_stamps.argtypes = [ctypes.c_void_p]
L.gp_debug_stamps.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda", 0)
flush = torch.ones(128 << 20, device=dev)
for shape in [(8, 1024, 768), (64, 256, 56, 56)]:
    x = torch.randn(shape, device=dev).reshape(-1)
    d = x.numel()
    for r in (10, 100):
        k = P.select_k(d, r)
        p = P.topk_compress(x, r)
        out = torch.empty(d, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        dbg = torch.zeros(8 * 4096, dtype=torch.int64, device=dev)
        for label in ("cold", "warm"):
            if label == "cold":
                flush.sum()
            else:
                L.gp_topk_decompress_frame(p.frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            dbg.zero_()
            L.gp_debug_dec_stamps(dbg.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.gp_topk_decompress_frame(p.frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            L.gp_debug_dec_stamps(None)
            a = dbg.cpu().numpy().reshape(4096, 8)
            G = int((a[:, 0] > 0).sum())
            s = a[:G, :5].astype(np.int64)
            t0 = s[:, 0].min()
            rel = (s - t0) / 1e3
            print(f"{shape} r={r} {label}: G={G} event={e0.elapsed_time(e1) * 1e3:.2f}us  entry spread "
                  f"{rel[:, 0].max():.2f}  search {np.mean(s[:, 1] - s[:, 0]) / 1e3:.2f}/{np.max(s[:, 1] - s[:, 0]) / 1e3:.2f}"
                  f"  setup {np.mean(s[:, 2] - s[:, 1]) / 1e3:.2f}  tiles {np.mean(s[:, 3] - s[:, 2]) / 1e3:.2f}/"
                  f"{np.max(s[:, 3] - s[:, 2]) / 1e3:.2f}  end(max) {rel[:, 4].max():.2f}", flush=True)
