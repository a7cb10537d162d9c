"""Does interleaving each unit's decompress right after its compress (same stream)
beat the bench's phase order (all compresses, then all decompresses)?

    python scripts/interleave_probe.py [--streams 4] [--ctas 37]

The configs[1] workload as bench.py builds it (24 distinct inputs, LPT stream
assignment); every variant is one CUDA graph replayed after a 512 MB L2 flush.
A development probe: prints ms per step and GB/s for each variant.
"""
import argparse
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2410_12707_b200 import _lib  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--ctas", default="37")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    g = torch.Generator(device=dev).manual_seed(1234)
    units = []
    for shape in bench.SHAPES:
        for kind in bench.KINDS:
            for r in bench.RATIOS:
                base = torch.randn(shape, device=dev, generator=g)
                x = (torch.relu(base) if kind == "activation" else base * 1e-3).reshape(-1).contiguous()
                d = x.numel()
                k = bench.select_k(d, r)
                units.append({"x": x, "d": d, "k": k, "r": r, "frame": torch.empty(16 + 12 * k, dtype=torch.uint8,
                                                                                      device=dev),
                              "out": torch.empty(d, device=dev)})
    step_bytes = sum(bench.pair_bytes(u["d"], 4, u["k"]) for u in units)
    ns = args.streams
    load = [0.0] * ns
    per = [[] for _ in range(ns)]

    def cost(u):
        return u["d"] * (2.2 if u["r"] <= 10 else 1.0) + 4e6

    for i in sorted(range(len(units)), key=lambda i: -cost(units[i])):
        j = min(range(ns), key=lambda j: load[j])
        per[j].append(i)
        load[j] += cost(units[i])
    for j in range(1, ns, 2):
        per[j].reverse()
    wsb = max(L.gp_topk_workspace_bytes(u["d"], 0) for u in units)
    wss = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(ns)]
    main_s = torch.cuda.current_stream(dev)
    for w in wss:
        L.gp_workspace_init(w.data_ptr(), wsb, main_s.cuda_stream)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    sts = [torch.cuda.Stream(dev) for _ in range(ns)]
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)

    def comp(u, j, st, ctas):
        assert L.gp_topk_compress_frame_ctas(u["x"].data_ptr(), 0, u["d"], u["k"], u["frame"].data_ptr(),
                                             wss[j].data_ptr(), wsb, st.cuda_stream, ctas) == 0

    def dec(u, st):
        assert L.gp_topk_decompress_frame(u["frame"].data_ptr(), u["k"], u["d"], u["out"].data_ptr(), 0, 0,
                                          err.data_ptr(), st.cuda_stream) == 0

    def variant(order, ctas):
        def body():
            cur = torch.cuda.current_stream(dev)
            for st in sts:
                st.wait_stream(cur)
            if order == "phases":
                for j, lst in enumerate(per):
                    for i in lst:
                        comp(units[i], j, sts[j], ctas)
                for st in sts:
                    cur.wait_stream(st)
                for st in sts:
                    st.wait_stream(cur)
                for j, lst in enumerate(per):
                    for i in lst:
                        dec(units[i], sts[j])
            else:  # interleaved: each unit's decompress right after its compress
                for j, lst in enumerate(per):
                    for i in lst:
                        comp(units[i], j, sts[j], ctas)
                        dec(units[i], sts[j])
            for st in sts:
                cur.wait_stream(st)
        body()
        torch.cuda.synchronize(dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(main_s)
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=side):
            body()
        ts = []
        for i in range(13):
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            gph.replay()
            e1.record(main_s)
            e1.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        assert int(err.item()) == 0
        t = statistics.median(ts)
        print(f"{order:12s} ctas={ctas:3d} streams={ns}: {t:.4f} ms/step  {step_bytes / t / 1e6:8.1f} GB/s", flush=True)

    for ctas in [int(c) for c in args.ctas.split(",")]:
        variant("phases", ctas)
        variant("interleaved", ctas)


if __name__ == "__main__":
    main()
