"""Decompress a frame that lives on another GPU (read over NVLink in place) -- timing and stage stamps.

    python scripts/remote_dec_probe.py       (needs 2 GPUs)

The frame is compressed on cuda:1; cuda:0 decompresses it (a) from a local
copy and (b) in place over NVLink (mode 2 trusted, mode 0 checked).  Prints
per-launch event times and the per-CTA stage stamps (search / tiles) of each.
(A deep-prefetch variant of the tiled kernel, cp.async rings of 4 batches per
thread, measured slower than (b) and was dropped.)
"""
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


def enable_peer(a, b):
    rt = ctypes.CDLL("libcudart.so.12")
    cur = ctypes.c_int()
    rt.cudaGetDevice(ctypes.byref(cur))
    rt.cudaSetDevice(a)
    r = rt.cudaDeviceEnablePeerAccess(b, 0)
    rt.cudaSetDevice(cur.value)
    return r


def main():
    print("enable peer 0->1:", enable_peer(0, 1), flush=True)
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    flush = torch.ones(128 << 20, device=d0)
    for shape in [(64, 256, 56, 56), (64, 1024, 14, 14)]:
        for r in (10, 100, 1000):
            with torch.cuda.device(d1):
                x = torch.relu(torch.randn(shape, device=d1)).reshape(-1)
                p = P.topk_compress(x, r)
                torch.cuda.synchronize(d1)
            d, k = x.numel(), p.k
            remote = p.frame
            local = remote.to(d0)
            ref = None
            with torch.cuda.device(d0):
                out = torch.empty(d, device=d0)
                err = torch.zeros(1, dtype=torch.int32, device=d0)
                dbg = torch.zeros(8 * 4096, dtype=torch.int64, device=d0)
                st = torch.cuda.current_stream(d0).cuda_stream
                for tag, fr, mode in (("local m2", local, 2), ("remote m2", remote, 2), ("remote m0", remote, 0)):
                    ts = []
                    for it in range(4):
                        flush.sum()
                        torch.cuda.synchronize(d0)
                        if it == 3:
                            dbg.zero_()
                            L.gp_debug_dec_stamps(dbg.data_ptr())
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        assert L.gp_topk_decompress_frame(fr.data_ptr(), k, d, out.data_ptr(), 0, mode, err.data_ptr(), st) == 0
                        e1.record()
                        torch.cuda.synchronize(d0)
                        L.gp_debug_dec_stamps(None)
                        ts.append(e0.elapsed_time(e1) * 1e3)
                    assert int(err.item()) == 0, (tag, int(err.item()))
                    if ref is None:
                        ref = out.clone()
                    same = torch.equal(out.view(torch.int32), ref.view(torch.int32))
                    a = dbg.cpu().numpy().reshape(4096, 8)
                    G = int((a[:, 0] > 0).sum())
                    s = a[:G, :5].astype(np.int64)
                    if G:
                        t0 = s[:, 0].min()
                        rel = (s - t0) / 1e3
                        stg = (f"G={G} search {np.mean(s[:, 1] - s[:, 0]) / 1e3:.2f}/{np.max(s[:, 1] - s[:, 0]) / 1e3:.2f} "
                               f"tiles {np.mean(s[:, 3] - s[:, 2]) / 1e3:.2f}/{np.max(s[:, 3] - s[:, 2]) / 1e3:.2f} "
                               f"end {rel[:, 4].max():.2f}")
                    else:
                        stg = "(sparse kernel: no stamps)"
                    print(f"{shape} r={r} k={k} {tag:10s}: {min(ts):8.1f} us  same={same}  {stg}", flush=True)


if __name__ == "__main__":
    main()
