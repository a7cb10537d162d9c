"""configs[4]: compression microbench sweep — tensor size 1 MB..1 GB x ratio 1e-1..1e-4, fp32 and bf16.

    python scripts/sweep.py [--out profiles/sweep_r01.json] [--cpu-max-mb 16]

Per case: compress and decompress device time (CUDA graphs, each launch after a
512 MB L2 read flush, differenced against the flush alone), algorithmic GB/s
(d*s + 12k per launch) and the fraction of the measured HBM
peak; a size-independent check of every GPU result (k entries, strictly
increasing indices, every kept |x| >= every dropped |x|, round trip equals x on
the support); and, for sizes up to --cpu-max-mb, the reference algorithm (the
NumPy oracle port, one core: np.argsort(kind="stable") is single-threaded) on
the same input: the reference's own geopipe.compressor from baseline/_ref
(the oracle port where that install is absent).  Synthetic N(0,1) data.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402
from scripts.graph_timing import graph_time  # noqa: E402

SIZES_MB = [1, 4, 16, 64, 256, 1024]


def cpu_impl():
    """The reference's own compressor (geopipe.compressor from baseline/_ref), else the oracle port."""
    import bench

    return bench._cpu_impl()
RATIOS = [10, 100, 1000, 10000]


def peak_gbs():
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        j = json.loads(p.read_text())
        for key in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if key in j:
                return float(j[key])
        for v in j.values():
            if isinstance(v, dict) and "hbm_gbs" in v:
                return float(v["hbm_gbs"])
    except (OSError, ValueError):
        pass
    return 6549.1


def check(x, frame, k, d, out):
    idx = frame[16:16 + 8 * k].view(torch.int64)
    assert idx.numel() == k
    if k > 1:
        assert bool((idx[1:] > idx[:-1]).all())
    a = x.float().abs()
    kept = torch.zeros(d, dtype=torch.bool, device=x.device)
    kept[idx] = True
    if k < d:
        t_min = a[kept].min()
        assert float(t_min) >= float(a[~kept].max())
        # ties at the threshold go to the lower index (the reference's stable
        # argsort, compressor.py:91-93): every dropped element equal to the
        # threshold lies after every kept one
        eq_dropped = torch.nonzero((~kept) & (a == t_min)).reshape(-1)
        eq_kept = torch.nonzero(kept & (a == t_min)).reshape(-1)
        if eq_dropped.numel() and eq_kept.numel():
            assert int(eq_dropped.min()) > int(eq_kept.max())
    ref = torch.zeros_like(x)
    ref[idx] = x[idx]
    assert torch.equal(out, ref)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--cpu-max-mb", type=int, default=256)
    ap.add_argument("--sizes", default=",".join(map(str, SIZES_MB)))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    peak = peak_gbs()
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    rows = []
    for dt, code, esz in (("fp32", 0, 4), ("bf16", 1, 2)):
        for mb in [int(s) for s in args.sizes.split(",")]:
            d = (mb << 20) // esz
            g = torch.Generator(device=dev).manual_seed(mb)
            x = torch.randn(d, device=dev, generator=g)
            if dt == "bf16":
                x = x.to(torch.bfloat16)
            wsb = L.gp_topk_workspace_bytes(d, code)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            L.gp_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
            out = torch.empty(d, dtype=x.dtype, device=dev)
            err = torch.zeros(1, dtype=torch.int32, device=dev)
            host = x.float().cpu().numpy() if mb <= args.cpu_max_mb else None
            for r in RATIOS:
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

                n = 4 if mb >= 256 else 10
                t0 = graph_time([fl], n=n, reps=3)
                tc = graph_time([fl, comp], n=n, reps=3) - t0
                t1 = graph_time([fl, comp, dec], n=n, reps=3)
                td = t1 - (tc + t0)
                torch.cuda.synchronize()
                comp()
                dec()
                torch.cuda.synchronize()
                assert int(err.item()) == 0
                check(x, frame, k, d, out)
                alg = d * esz + 12 * k
                row = {"dtype": dt, "size_mb": mb, "d": d, "ratio": r, "k": k, "compress_us": round(tc, 2),
                       "decompress_us": round(td, 2), "compress_gbs": round(alg / tc / 1e3, 1),
                       "decompress_gbs": round(alg / td / 1e3, 1),
                       "pair_frac_of_peak": round(2 * alg / (tc + td) / 1e3 / peak, 4), "checked": True}
                if host is not None and dt == "fp32":
                    run, ckind, _ = cpu_impl()
                    t = time.perf_counter()
                    run(host, r)
                    dt_cpu = time.perf_counter() - t
                    row["cpu_reference_gbs"] = round(2 * alg / dt_cpu / 1e9, 4)
                    row["cpu_reference_s"] = round(dt_cpu, 3)
                    row["cpu_reference_kind"] = ckind
                    row["cpu_reference_cores"] = 1
                rows.append(row)
                print(json.dumps(row), flush=True)
            del ws, out
            torch.cuda.empty_cache()
    res = {"config": "configs[4]: compression microbench sweep (size 1 MB-1 GB x ratio 1e-1..1e-4, fp32 and bf16)",
           "timing": "CUDA graphs, each launch after a 512 MB L2 read flush, differenced; algorithmic bytes d*s+12k",
           "peak_gbs": peak, "cpu_reference": "the reference's geopipe.compressor (baseline/_ref; the oracle port "
           f"where absent), 1 core, fp32 sizes <= {args.cpu_max_mb} MB, compress+decompress of the same input",
           "data": "synthetic N(0,1)", "rows": rows}
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
