#!/usr/bin/env python
"""Small-size driver for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

Runs every kernel path through the C-ABI on cuda:0, each result checked bit for
bit against the oracle (so a run that "passes" the tool also computed the right
thing):

  compress   fast path (N(0,1)), slow path (massive ties: > 64K final
             candidates), rescan (ascending input: the top CTAs' watermarks sit
             above B1), bf16, fp64, unaligned input, k == d (keep-all kernel)
  capped     four concurrent capped-grid compresses on four streams
  decompress sparse fill+scatter kernel (r = 100), tiled TMA-store kernel (r = 10),
             residual mode, unsorted general scatter, out-of-range flag
  plan       the on-device Eq. 6 kernel

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [--small]
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import compressor_oracle as O  # noqa: E402  (the checker only)
from paper_2410_12707_b200 import _lib  # noqa: E402

SMALL = "--small" in sys.argv  # racecheck is ~100x slower: smaller tensors
DEV = torch.device("cuda", 0)
L = _lib.lib()


def select_k(d, r):
    return max(1, int(np.floor(d / r)))


def ws_for(d, dtype):
    n = L.gp_topk_workspace_bytes(d, dtype)
    ws = torch.empty(n, dtype=torch.uint8, device=DEV)
    assert L.gp_workspace_init(ws.data_ptr(), n, torch.cuda.current_stream(DEV).cuda_stream) == 0
    return ws, n


def compress_frame(x: torch.Tensor, ratio, dtype=0, ctas=0, stream=None, ws=None):
    d = x.numel()
    k = select_k(d, ratio)
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=DEV)
    if ws is None:
        ws = ws_for(d, dtype)
    st = (stream or torch.cuda.current_stream(DEV)).cuda_stream
    rc = L.gp_topk_compress_frame_ctas(x.data_ptr(), dtype, d, k, frame.data_ptr(), ws[0].data_ptr(), ws[1], st, ctas)
    assert rc == 0, rc
    return frame, k


def check_frame(name, host, ratio, frame):
    ref = O.compress_frame(host, ratio, method="threshold")
    got = frame.cpu().numpy().tobytes()
    assert got == ref, f"{name}: frame differs from the oracle"
    print(f"ok  compress {name}: d={host.size} r={ratio}", flush=True)


def main():
    g = torch.Generator(device=DEV).manual_seed(0)
    n = 300_000 if SMALL else 2_000_000
    cases = []
    x = torch.randn(n, device=DEV, generator=g)
    cases.append(("fast f32", x, 100.0))
    cases.append(("fast f32 r=10", x, 10.0))
    ties = torch.ones(n, device=DEV)
    ties[::7] = 2.0
    cases.append(("slow path (ties)", ties, 3.0))
    cases.append(("rescan (ascending)", torch.arange(n, device=DEV, dtype=torch.float32), 100.0))
    cases.append(("unaligned", x[3:3 + n // 2], 50.0))
    for name, t, r in cases:
        frame, _ = compress_frame(t.contiguous() if name != "unaligned" else t, r)
        check_frame(name, t.cpu().numpy(), r, frame)
    # bf16 and fp64
    xb = x.to(torch.bfloat16)
    fb, _ = compress_frame(xb, 100.0, dtype=1)
    check_frame("bf16", xb.float().cpu().numpy(), 100.0, fb)
    xd = x.double()[: n // 4]
    fd, _ = compress_frame(xd, 100.0, dtype=2)
    check_frame("f64", xd.cpu().numpy(), 100.0, fd)
    fa, _ = compress_frame(x[:1000].contiguous(), 1.0)
    check_frame("keep-all", x[:1000].cpu().numpy(), 1.0, fa)

    # the single-cluster kernel (gp_cluster.cu): default-routed short vectors,
    # and every vector that fits one cluster (mode 2), incl. ties, unaligned, bf16, fp64
    for name, t, r, dt in (("cluster f32 (default route)", x[:90_000].contiguous(), 10.0, 0),
                           ("cluster f32 tail", x[:33].contiguous(), 3.0, 0)):
        fr, _ = compress_frame(t, r, dtype=dt)
        check_frame(name, t.cpu().numpy(), r, fr)
    prev = L.gp_set_cluster_path(2)
    for name, t, r, dt in (("cluster f32", x[:n].contiguous() if n <= 393_216 else x[:380_000].contiguous(), 100.0, 0),
                           ("cluster ties", ties[:200_000].contiguous(), 3.0, 0),
                           ("cluster unaligned", x[5:5 + 100_000], 10.0, 0),
                           ("cluster bf16", xb[:300_000].contiguous(), 10.0, 1),
                           ("cluster f64", x.double()[:200_000].contiguous(), 100.0, 2)):
        fr, _ = compress_frame(t, r, dtype=dt)
        check_frame(name, (t.float() if dt == 1 else t).cpu().numpy(), r, fr)
    L.gp_set_cluster_path(prev)

    # four concurrent capped grids, a workspace per stream
    sts = [torch.cuda.Stream(DEV) for _ in range(4)]
    xs = [torch.randn(n, device=DEV, generator=g) for _ in range(4)]
    wss = [ws_for(n, 0) for _ in range(4)]
    torch.cuda.synchronize(DEV)
    outs = []
    for i, (st, xi, w) in enumerate(zip(sts, xs, wss)):
        outs.append(compress_frame(xi, [10.0, 100.0, 1000.0, 100.0][i], ctas=37, stream=st, ws=w)[0])
    torch.cuda.synchronize(DEV)
    for i, (xi, f) in enumerate(zip(xs, outs)):
        check_frame(f"capped grid stream {i}", xi.cpu().numpy(), [10.0, 100.0, 1000.0, 100.0][i], f)

    # decompress: sparse kernel (r=100), tiled TMA-store kernel (r=10), residual
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    host = x.cpu().numpy()
    for r in (100.0, 10.0):
        frame, k = compress_frame(x, r)
        out = torch.empty(n, device=DEV)
        assert L.gp_topk_decompress_frame(frame.data_ptr(), k, n, out.data_ptr(), 0, 0, err.data_ptr(),
                                          torch.cuda.current_stream(DEV).cuda_stream) == 0
        vals, idx, d = O.from_bytes(frame.cpu().numpy().tobytes())
        ref = O.topk_decompress(vals.astype(np.float32), idx, d)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32)), f"decompress r={r}"
        base = torch.randn(n, device=DEV, generator=g)
        acc = base.clone()
        assert L.gp_topk_decompress_frame(frame.data_ptr(), k, n, acc.data_ptr(), 0, 1, err.data_ptr(),
                                          torch.cuda.current_stream(DEV).cuda_stream) == 0
        exp = base.cpu().numpy().copy()
        exp[idx] += vals.astype(np.float32)
        assert np.array_equal(acc.cpu().numpy(), exp), f"residual r={r}"
        assert int(err.item()) == 0
        print(f"ok  decompress r={r} (zero + residual)", flush=True)
    # unsorted general scatter (numpy last-write-wins) and the out-of-range flag
    d = 10_000
    idx = torch.tensor([5, 3, 5, 9999, 0], dtype=torch.int64, device=DEV)
    vals = torch.tensor([1.0, 2.0, 3.0, 4.0, 5.0], device=DEV)
    out = torch.empty(d, device=DEV)
    scratch = torch.empty(d, dtype=torch.int32, device=DEV)
    assert L.gp_topk_decompress_unsorted(idx.data_ptr(), 8, vals.data_ptr(), 0, 5, d, out.data_ptr(), 0,
                                         scratch.data_ptr(), err.data_ptr(),
                                         torch.cuda.current_stream(DEV).cuda_stream) == 0
    exp = np.zeros(d, np.float32)
    exp[idx.cpu().numpy()] = vals.cpu().numpy()
    assert np.array_equal(out.cpu().numpy(), exp) and int(err.item()) == 0
    bad = torch.tensor([1, 2, d + 5], dtype=torch.int64, device=DEV)
    assert L.gp_topk_decompress(bad.data_ptr(), 8, vals.data_ptr(), 0, 3, d, out.data_ptr(), 0, 0, err.data_ptr(),
                                torch.cuda.current_stream(DEV).cuda_stream) == 0
    assert int(err.item()) & _lib.FLAG_OUT_OF_RANGE
    err.zero_()
    print("ok  decompress unsorted + out-of-range flag", flush=True)

    # on-device Eq. 6
    import paper_2410_12707_b200 as P
    R = torch.tensor([10.0, 5.0, 1.0], dtype=torch.float64, device=DEV)
    r, kk, status = P.adatopk_plan_device(R, 100.0, torch.full((3,), 6_553_600, dtype=torch.int64, device=DEV))
    assert int(status.item()) == 0 and r.tolist() == [300.0, 150.0, 30.0], r.tolist()
    print("ok  plan kernel", flush=True)
    torch.cuda.synchronize(DEV)
    print("ALL CASES OK")


if __name__ == "__main__":
    main()
