"""CUDA-event timing of compress / decompress launches + per-stage breakdown (development aid)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402

STAGES = ["entry->sample", "sample->stream", "stream->B1arr", "B1", "stage2", "split+fc", "B2", "fc-resolve", "walk"]


def cold_times(fn, flush, reps=30):
    ts = []
    for _ in range(reps):
        flush.sum()  # read-only flush: L2 ends full of clean lines
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def warm_time(fn, n=100):
    fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) * 1e3 / n


def main():
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    L.gp_debug_stamps.argtypes = [ctypes.c_void_p]
    L.gp_debug_stamps.restype = None
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)  # 512 MB
    st = torch.cuda.current_stream().cuda_stream
    dbg = torch.zeros(1024 * 32, dtype=torch.int64, device=dev)
    shapes = [("C1 gpt2-small 8x1024x768", (8, 1024, 768)), ("C3 gpt2-med 8x1024x1024", (8, 1024, 1024)),
              ("resnet 64x2048x7x7", (64, 2048, 7, 7)), ("resnet 64x256x56x56", (64, 256, 56, 56))]
    g = torch.Generator(device=dev).manual_seed(0)
    for name, shape in shapes:
        x = torch.randn(shape, device=dev, generator=g).reshape(-1)
        d = x.numel()
        for r in (10, 100, 1000):
            k = P.select_k(d, r)
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
            wsb = L.gp_topk_workspace_bytes(d, 0)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            L.gp_workspace_init(ws.data_ptr(), wsb, st)
            out = torch.empty(d, device=dev)
            err = torch.zeros(1, dtype=torch.int32, device=dev)

            def comp():
                assert L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, st) == 0

            def decomp():
                assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(), st) == 0

            for _ in range(3):
                comp()
                decomp()
            tc = cold_times(comp, flush)
            td = cold_times(decomp, flush)
            wc = warm_time(comp)
            wd = warm_time(decomp)
            byts = d * 4 + k * 12
            print(f"{name:26s} r={r:5d} d={d:9d} k={k:8d} | compress cold {tc:7.2f} us ({byts / tc / 1e3:6.0f} GB/s)"
                  f" warm {wc:7.2f} | decompress cold {td:7.2f} us ({byts / td / 1e3:6.0f} GB/s) warm {wd:7.2f}",
                  flush=True)
            # stage breakdown of one cold launch
            dbg.zero_()
            L.gp_debug_stamps(dbg.data_ptr())
            flush.sum()
            comp()
            torch.cuda.synchronize()
            L.gp_debug_stamps(None)
            a = dbg.cpu().numpy().reshape(1024, 32)
            G = int((a[:, 0] > 0).sum())
            ns = a[:G, :9].astype(np.int64)
            t0 = ns[:, 0].min()
            parts = []
            for i in range(1, 9):
                delta = ns[:, i] - ns[:, i - 1]
                parts.append(f"{STAGES[i]}={np.mean(delta) / 1e3:.2f}/{np.max(delta) / 1e3:.2f}")
            print(f"    G={G} entry-skew={(ns[:, 0].max() - t0) / 1e3:.2f}us total(max end)={(ns[:, 8].max() - t0) / 1e3:.2f}us "
                  + " ".join(parts), flush=True)


if __name__ == "__main__":
    main()
