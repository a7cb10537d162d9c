"""Per-kernel device time of compress / decompress inside CUDA graphs (development aid).

Each measurement replays a graph of N iterations; per-op time is the difference
between graphs with and without the op, so CPU launch latency is excluded and
every op starts cold (a 512 MB read flushes L2 between iterations).
"""
import ctypes
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402

STAGES = ["watermark", "stream", "flush+B1", "find-B1", "split+fc", "B2", "fc-resolve", "walk"]


def graph_time(fns, n=20, reps=7):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            for f in fns:
                f()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n)
    return statistics.median(ts)


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    L = _lib.lib()
    L.gp_debug_stamps.argtypes = [ctypes.c_void_p]
    L.gp_debug_stamps.restype = None
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)  # 512 MB read
    dbg = torch.zeros(1024 * 32, dtype=torch.int64, device=dev)
    peak = 6549.1
    shapes = [("C1 gpt2-small 8x1024x768", (8, 1024, 768), "f32"), ("C3 gpt2-med 8x1024x1024", (8, 1024, 1024), "f32"),
              ("resnet 64x2048x7x7", (64, 2048, 7, 7), "f32"), ("resnet 64x512x28x28", (64, 512, 28, 28), "f32"),
              ("resnet 64x256x56x56", (64, 256, 56, 56), "f32"), ("C3 bf16 8x1024x1024", (8, 1024, 1024), "bf16")]
    ratios = [10, 100, 1000] if len(sys.argv) < 2 else [float(r) for r in sys.argv[1].split(",")]
    if os.environ.get("GT_SHAPES"):  # comma-separated substrings of the shape names
        keep = os.environ["GT_SHAPES"].split(",")
        shapes = [s for s in shapes if any(k in s[0] for k in keep)]
    g = torch.Generator(device=dev).manual_seed(0)
    for name, shape, dt in shapes:
        x = torch.randn(shape, device=dev, generator=g).reshape(-1)
        code, esz = 0, 4
        if dt == "bf16":
            x, code, esz = x.to(torch.bfloat16), 1, 2
        d = x.numel()
        for r in ratios:
            k = P.select_k(d, r)
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
            wsb = L.gp_topk_workspace_bytes(d, code)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            L.gp_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
            out = torch.empty(d, dtype=x.dtype, device=dev)
            err = torch.zeros(1, dtype=torch.int32, device=dev)

            def fl():
                flush.sum()
                if os.environ.get("GT_REINIT"):  # exit-at-phase variants skip the workspace cleanup
                    L.gp_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)

            def comp():
                st = torch.cuda.current_stream().cuda_stream
                assert L.gp_topk_compress_frame(x.data_ptr(), code, d, k, frame.data_ptr(), ws.data_ptr(), wsb, st) == 0

            def decomp():
                st = torch.cuda.current_stream().cuda_stream
                assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), code, 0, err.data_ptr(),
                                                  st) == 0

            t0 = graph_time([fl])
            t1 = graph_time([fl, comp])
            if os.environ.get("GT_COMPRESS_ONLY"):  # exit-at-phase variants: no valid frame to decompress
                tw = graph_time([comp])
                print(f"{name:26s} r={r:6g} k={k:8d} | compress {t1 - t0:7.2f} us (warm {tw:6.2f})", flush=True)
                continue
            t2 = graph_time([fl, comp, decomp])
            tw = graph_time([comp])
            twd = graph_time([decomp])
            tsl = graph_time([fl, lambda: torch.cuda._sleep(1)]) - t0
            tc, td = t1 - t0, t2 - t1
            cb = d * esz + 12 * k
            print(f"{name:26s} r={r:6g} k={k:8d} | compress {tc:7.2f} us {cb / tc / 1e3:6.0f} GB/s"
                  f" (warm {tw:6.2f}) | decompress {td:7.2f} us {cb / td / 1e3:6.0f} GB/s (warm {twd:6.2f}) | cold tiny kernel {tsl:5.2f} | pair {tc + td:7.2f} us"
                  f" = {2 * cb / (tc + td) / 1e3 / peak * 100:5.1f}% of {peak:.0f} GB/s", flush=True)
            for label in ("cold", "warm"):
                if label == "cold":
                    flush.sum()
                else:
                    comp()
                torch.cuda.synchronize()
                dbg.zero_()
                L.gp_debug_stamps(dbg.data_ptr())
                comp()
                torch.cuda.synchronize()
                L.gp_debug_stamps(None)
                a = dbg.cpu().numpy().reshape(1024, 32)
                G = int((a[:, 0] > 0).sum())
                ns = a[:G, :9].astype(np.int64)
                t00 = ns[:, 0].min()
                parts = []
                for i in range(1, 9):
                    delta = ns[:, i] - ns[:, i - 1]
                    if (ns[:, i] > 0).all():
                        parts.append(f"{STAGES[i - 1]}={np.mean(delta) / 1e3:.2f}/{np.max(delta) / 1e3:.2f}")
                print(f"    {label} G={G} skew={(ns[:, 0].max() - t00) / 1e3:.2f} "
                      f"end={(ns[:, 8].max() - t00) / 1e3:.2f}us " + " ".join(parts), flush=True)
                sub = a[:G, :11].astype(np.int64)
                if (sub[:, 9] > 0).all() and (sub[:, 10] > 0).all():  # fast-path stage-3 split (stamps 9, 10)
                    print(f"      stage3: gather={np.mean(sub[:, 9] - sub[:, 6]) / 1e3:.2f} "
                          f"select={np.mean(sub[:, 7] - sub[:, 9]) / 1e3:.2f} "
                          f"prefix={np.mean(sub[:, 10] - sub[:, 7]) / 1e3:.2f} "
                          f"walk={np.mean(sub[:, 8] - sub[:, 10]) / 1e3:.2f}", flush=True)


if __name__ == "__main__":
    main()
