"""GPU parity at the remaining BASELINE shapes, the frame checks on the wire
path, the standalone frame pack/unpack, and device-resident k.

Bar: bit-exact against the oracle (integer/byte/index work), the oracle being
pinned to frames the reference itself produced (tests/test_oracle_golden.py).
"""
import dataclasses

import numpy as np
import pytest
import torch

import paper_2410_12707_b200 as P
from paper_2410_12707_b200 import _lib
from paper_2410_12707_b200 import pipeline as PL
from paper_2410_12707_b200.transport import FrameCodec
from oracle import compressor_oracle as O

pytestmark = pytest.mark.gpu


def _check(x: torch.Tensor, ratio: float):
    """Frame and decompressed tensor bit-exact against the oracle."""
    p = P.topk_compress(x, ratio)
    host = x.float().cpu().numpy().reshape(-1) if x.dtype == torch.bfloat16 else x.cpu().numpy().reshape(-1)
    frame = O.compress_frame(host, ratio, method="threshold")
    assert p.to_bytes() == frame, f"frame differs at r={ratio}"
    dense = P.topk_decompress(p)
    vals, idx, d = O.from_bytes(frame)
    ref = O.topk_decompress(vals.astype(np.float32), idx, d)
    assert np.array_equal(dense.cpu().numpy().view(np.uint32), ref.view(np.uint32)), f"decompress r={ratio}"
    return p


# --------------------------------------------------------------------------- BASELINE shapes


@pytest.mark.parametrize("ratio", [100.0, 300.0])
def test_c3_gpt2_medium_fp32_vs_oracle(cuda, ratio):
    """configs[2]: the GPT-2 medium boundary [8,1024,1024] fp32 (d = 8,388,608)."""
    g = torch.Generator(device=cuda).manual_seed(31)
    _check(torch.randn(8, 1024, 1024, device=cuda, generator=g), ratio)


def test_c4_gpt2_xl_fp32_at_every_plan_ratio(cuda):
    """configs[3]: [4,1024,1600] fp32 at every ratio the 8-stage Eq. 6 plan over
    the two-cluster link model produces (3r on the slow link, the fast links'
    ratios clamped at 1 by max(1, .))."""
    d = 4 * 1024 * 1600
    plan = PL.link_plan(8, "adatopk", 100.0, PL.two_cluster_link_times(8, 4 * d))
    ratios = sorted(set(plan.per_link.values()))
    assert 300.0 in ratios
    g = torch.Generator(device=cuda).manual_seed(32)
    x = torch.randn(4, 1024, 1600, device=cuda, generator=g)
    grad = torch.randn(4, 1024, 1600, device=cuda, generator=g) * 1e-4
    for r in ratios:
        if r <= 1.0:  # the executor passes these through dense (executor.py:210-212)
            continue
        _check(x, r)
        _check(grad, r)


@pytest.mark.parametrize("kind", ["activation", "gradient"])
def test_resnet101_largest_boundary_vs_oracle(cuda, kind):
    """configs[1]'s largest boundary [64,256,56,56] (d = 51,380,224) at every
    ratio, bit-exact against the oracle (about 2 s of numpy per ratio)."""
    g = torch.Generator(device=cuda).manual_seed(33)
    x = torch.randn(64, 256, 56, 56, device=cuda, generator=g)
    x = torch.relu(x) if kind == "activation" else x * 1e-3
    for r in (10.0, 100.0, 1000.0):
        _check(x, r)


# --------------------------------------------------------------------------- the wire path's checks


def test_frame_codec_flags_corrupt_frames(cuda):
    """A received frame whose header disagrees with the receiver's (d, k), or
    holds an index outside [0, d), raises at the step's flag check."""
    codec = FrameCodec(cuda)
    x = torch.randn(100_000, device=cuda)
    out = torch.empty_like(x)
    frame = codec.compress(x, 10.0)
    codec.decompress(frame, out, 10.0)
    codec.check()  # a good frame
    with pytest.raises(ValueError, match="header"):
        codec.decompress(frame, out, 20.0)  # the receiver expects k = 5000
        codec.check()
    assert int(torch.count_nonzero(out)) == 0  # nothing scattered from a mismatched frame
    bad = frame.clone()
    bad[16:16 + 8 * 10000].view(torch.int64)[-1] = 10 ** 7  # still increasing, past d
    codec.decompress(bad, out, 10.0)
    with pytest.raises(P.IndexOutOfRange):
        codec.check()
    unsorted = frame.clone()
    iv = unsorted[16:16 + 8 * 10000].view(torch.int64)
    iv[5], iv[6] = iv[6].clone(), iv[5].clone()
    codec.decompress(unsorted, out, 10.0)
    with pytest.raises(ValueError, match="increasing"):
        codec.check()
    codec.check()  # the flag was cleared


def test_accumulate_with_unsorted_indices_raises(cuda):
    vals = torch.ones(3, device=cuda)
    p = P.SparsePayload(values=vals, indices=torch.tensor([5, 2, 9], device=cuda), original_len=10)
    with pytest.raises(ValueError):
        P.topk_decompress(p, out=torch.zeros(10, device=cuda), accumulate=True)
    dense = P.topk_decompress(p)  # zero mode: numpy's last-write-wins general scatter
    assert dense.tolist() == [0, 0, 1, 0, 0, 1, 0, 0, 0, 1]


def test_payload_length_mismatch_raises(cuda):
    p = P.SparsePayload(values=torch.ones(4, device=cuda), indices=torch.tensor([1, 2, 3], device=cuda),
                        original_len=10)
    with pytest.raises(ValueError):
        P.topk_decompress(p)
    q = P.topk_compress(torch.randn(1000, device=cuda), 10)
    with pytest.raises(ValueError):
        P.topk_decompress(dataclasses.replace(q, values=q.values[:-1]))
    raw = q.to_bytes()
    with pytest.raises(ValueError):
        P.SparsePayload.from_bytes(raw[:-4])


def test_to_bytes_serialises_the_current_fields(cuda):
    """to_bytes() returns the cached device frame only while the payload is
    unmodified; in-place edits, replaced fields and bf16/f64 payloads are packed
    on the device (gp_pack_frame) from the fields as they are now."""
    x = torch.randn(50_000, device=cuda)
    p = P.topk_compress(x, 10)
    assert p.to_bytes() == O.compress_frame(x.cpu().numpy(), 10, method="threshold")
    vals, idx, d = p.values.cpu().numpy(), p.indices.cpu().numpy(), p.original_len
    q = P.topk_compress(x.to(torch.bfloat16), 10)
    q.values[3] = 7.0  # a bf16 tensor separate from the frame
    want = O.to_bytes(q.values.float().cpu().numpy(), q.indices.cpu().numpy(), d)
    assert q.to_bytes() == want
    r = dataclasses.replace(p, values=p.values * 2)
    assert r.to_bytes() == O.to_bytes(vals * 2, idx, d)
    s = P.topk_compress(x.double(), 10)
    assert s.to_bytes() == O.compress_frame(x.double().cpu().numpy(), 10, method="threshold")
    s.original_len = d + 5
    assert s.to_bytes()[:8] == np.array([d + 5], dtype="<u8").tobytes()
    f = P.SparsePayload.from_bytes(p.to_bytes(), device=cuda)
    assert f.values.dtype == torch.float64 and f.to_bytes() == p.to_bytes()
    f.values[0] = 1.5
    assert f.to_bytes() != p.to_bytes()


def test_pack_unpack_frame_cabi(cuda):
    L = _lib.lib()
    rng = np.random.default_rng(5)
    d, k = 1_000_003, 4097
    idx = np.sort(rng.choice(d, k, replace=False)).astype(np.int64)
    vals = rng.standard_normal(k)
    sp = torch.cuda.current_stream().cuda_stream
    for vdt, code in ((torch.float32, 0), (torch.bfloat16, 1), (torch.float64, 2)):
        v = torch.from_numpy(vals).to(vdt).to(cuda)
        for ib in (8, 4):
            it = torch.from_numpy(idx.astype(np.int64 if ib == 8 else np.int32)).to(cuda)
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda)
            assert L.gp_pack_frame(it.data_ptr(), ib, v.data_ptr(), code, k, d, frame.data_ptr(), sp) == 0
            want = O.to_bytes(v.float().cpu().numpy() if vdt != torch.float64 else v.cpu().numpy(), idx, d)
            assert frame.cpu().numpy().tobytes() == want, (vdt, ib)
    # unpack: values widened to f64 (the reference from_bytes), header read on the device
    frame = torch.frombuffer(bytearray(O.to_bytes(vals.astype(np.float32), idx, d)), dtype=torch.uint8).to(cuda)
    oi = torch.empty(k, dtype=torch.int64, device=cuda)
    ov = torch.empty(k, dtype=torch.float64, device=cuda)
    hdr = torch.empty(2, dtype=torch.int64, device=cuda)
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    assert L.gp_unpack_frame(frame.data_ptr(), k, d, oi.data_ptr(), ov.data_ptr(), 2, hdr.data_ptr(), err.data_ptr(),
                             sp) == 0
    assert hdr.tolist() == [d, k] and int(err.item()) == 0
    assert np.array_equal(oi.cpu().numpy(), idx)
    assert np.array_equal(ov.cpu().numpy(), vals.astype(np.float32).astype(np.float64))
    assert L.gp_unpack_frame(frame.data_ptr(), k - 1, d, oi.data_ptr(), ov.data_ptr(), 2, None, err.data_ptr(),
                             sp) == 0
    assert int(err.item()) == _lib.FLAG_HEADER  # k above the capacity


# --------------------------------------------------------------------------- device-resident k


def test_device_k_replans_every_step_without_host_sync(cuda):
    """north_star item 4: per-link k from Eq. 6 on the device, read by the
    compress kernel from device memory; the receiver reads k from the frame
    header.  Five re-plans with different link times under
    torch.cuda.set_sync_debug_mode("error") (any host sync would raise), then
    every frame and every decompressed tensor is checked against the oracle
    applied with the reference's plan (compressor.py:111-129, :73-76)."""
    d, base = 6_553_600 // 4, 100.0
    links = [(0, 1), (1, 2), (2, 3), (1, 0), (2, 1), (3, 2)]
    plan = PL.DevicePlan(links, d, base, cuda, ratio_floor=1.0)  # k_cap = d: never clamps
    codec = FrameCodec(cuda)
    rng = np.random.default_rng(0)
    R_host = [rng.uniform(1e-4, 1e-2, len(links)) for _ in range(5)]
    R_dev = torch.tensor(np.array(R_host), dtype=torch.float64, device=cuda)
    g = torch.Generator(device=cuda).manual_seed(40)
    xs = [torch.randn(d, device=cuda, generator=g) for _ in range(2)]
    k_cap = plan.k_cap
    frames, outs = [], []
    torch.cuda.synchronize()
    torch.cuda.set_sync_debug_mode("error")
    try:
        for step in range(5):
            plan.replan(R_dev[step])
            for li in (0, 4):  # one FP and one BP link per step
                f = codec.compress_dk(xs[li % 2], plan.k_slot(links[li]), k_cap)
                o = torch.empty(d, device=cuda)
                codec.decompress_dk(f, o, k_cap)
                frames.append((step, li, f))
                outs.append(o)
    finally:
        torch.cuda.set_sync_debug_mode(0)
    torch.cuda.synchronize()
    codec.check()
    assert int(plan.clamped.item()) == 0
    for (step, li, f), o in zip(frames, outs):
        r = O.adatopk_ratios({lk: v for lk, v in zip(links, R_host[step])}, base)[links[li]]
        k = O.select_k(d, r)
        want = O.compress_frame(xs[li % 2].cpu().numpy(), r, method="threshold")
        assert f[: 16 + 12 * k].cpu().numpy().tobytes() == want, (step, li)
        vals, idx, _ = O.from_bytes(want)
        ref = O.topk_decompress(vals.astype(np.float32), idx, d)
        assert np.array_equal(o.cpu().numpy().view(np.uint32), ref.view(np.uint32)), (step, li)


def test_device_k_edge_cases(cuda):
    """k == d keeps every element (ratio <= 1: the executor's dense pass-through,
    bit for bit); k outside [1, k_cap] raises GP_FLAG_BAD_K on the sender and the
    receiver flags the invalid header and scatters nothing."""
    codec = FrameCodec(cuda)
    x = torch.randn(70_001, device=cuda)
    x[7] = float("nan")
    x[9] = -0.0
    d = x.numel()
    kd = torch.tensor([d], dtype=torch.int64, device=cuda)
    f = codec.compress_dk(x, kd, d)
    out = torch.empty_like(x)
    codec.decompress_dk(f, out, d)
    codec.check()
    assert torch.equal(out.view(torch.int32), x.view(torch.int32))
    for bad in (0, 101):
        kb = torch.tensor([bad], dtype=torch.int64, device=cuda)
        f = codec.compress_dk(x, kb, 100)
        with pytest.raises(ValueError, match="k outside"):
            codec.check()
        out.fill_(1.0)
        codec.decompress_dk(f, out, 100)
        with pytest.raises(ValueError, match="header"):
            codec.check()
        assert int(torch.count_nonzero(out)) == 0


def test_one_workspace_serves_every_fitting_call(cuda):
    """One C-ABI workspace, zeroed once, sized for the largest vector, then
    calls of every size and dtype in an order that shrinks and grows d (the
    bench's per-stream pattern): every frame stays bit-exact, so no call's
    per-call regions overwrite the state a later call relies on."""
    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(41)
    sizes = [6_000_000, 1000, 3_000_001, 17, 6_000_000, 250_000, 4_000_000]
    wsb = max(L.gp_topk_workspace_bytes(n, dt) for n in sizes for dt in (0, 1, 2))
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda)
    sp = torch.cuda.current_stream().cuda_stream
    assert L.gp_workspace_init(ws.data_ptr(), wsb, sp) == 0
    for rep in range(2):
        for i, n in enumerate(sizes):
            for dt, tdt in ((0, torch.float32), (1, torch.bfloat16), (2, torch.float64)):
                if dt == 2 and n > 1_000_000:
                    continue
                x = torch.randn(n, device=cuda, generator=g).to(tdt)
                r = (3.0, 10.0, 100.0, 1000.0)[(i + rep + dt) % 4]
                k = O.select_k(n, r)
                frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda)
                assert L.gp_topk_compress_frame(x.data_ptr(), dt, n, k, frame.data_ptr(), ws.data_ptr(), wsb, sp) == 0
                host = x.float().cpu().numpy() if dt == 1 else x.cpu().numpy()
                assert frame.cpu().numpy().tobytes() == O.compress_frame(host, r, method="threshold"), (rep, n, dt, r)


def test_opdata_envelope_device(cuda):
    """Envelope written and checked by stream-ordered kernels (fields passed by
    value); a mismatch raises GP_FLAG_ENVELOPE, read at the step's flag check."""
    from paper_2410_12707_b200 import transport as T

    codec = FrameCodec(cuda)
    f = T.envelope_fields(7, 2, 0, 1, T.KIND_ACTIVATION, True, 4096, (8, 1024, 768))
    buf = torch.empty(T.ENVELOPE_BYTES + 64, dtype=torch.uint8, device=cuda)
    T.write_envelope(buf, f)
    assert buf[:T.ENVELOPE_BYTES].view(torch.int64).tolist() == f
    T.check_envelope(buf, f, codec.err)
    codec.check()
    T.check_envelope(buf, T.envelope_fields(7, 3, 0, 1, T.KIND_ACTIVATION, True, 4096, (8, 1024, 768)), codec.err)
    with pytest.raises(ValueError, match="envelope"):
        codec.check()


@pytest.mark.parametrize("ratio", [3.0, 10.0, 100.0])
def test_trusted_decompress_equals_checked(cuda, ratio):
    """GP_DECOMPRESS_TRUSTED (a frame gp_topk_compress just wrote: strictly
    increasing by construction) skips only the O(k) sortedness scan: the output
    is bit-identical to the checked decompress, in zero and residual mode, and a
    frame with an out-of-range index is still flagged (the range check stays)."""
    L = _lib.lib()
    codec = FrameCodec(cuda)
    g = torch.Generator(device=cuda).manual_seed(50)
    x = torch.randn(3_000_017, device=cuda, generator=g)
    d, k = x.numel(), O.select_k(x.numel(), ratio)
    frame = codec.compress(x, ratio)
    sp = torch.cuda.current_stream().cuda_stream
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    base = torch.randn(d, device=cuda, generator=g)
    for mode in (0, 1):
        a, b = base.clone(), base.clone()
        assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, a.data_ptr(), 0, mode, err.data_ptr(), sp) == 0
        assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, b.data_ptr(), 0, mode | 2, err.data_ptr(), sp) == 0
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)) and int(err.item()) == 0
    bad = frame.clone()
    bad[16:16 + 8 * k].view(torch.int64)[-1] = d + 7
    assert L.gp_topk_decompress_frame(bad.data_ptr(), k, d, base.data_ptr(), 0, 2, err.data_ptr(), sp) == 0
    assert int(err.item()) & _lib.FLAG_OUT_OF_RANGE
    p = P.topk_compress(x, ratio)  # the drop-in: kernel-made payloads decompress trusted, no host sync
    ref = torch.zeros_like(x)
    ref[p.indices] = x[p.indices]
    assert torch.equal(P.topk_decompress(p).view(torch.int32), ref.view(torch.int32))


# --------------------------------------------------------------------------- input dtypes


@pytest.mark.parametrize("dtype", [np.int64, np.int32, np.int16, np.float16])
def test_input_dtype_is_kept_like_the_reference(cuda, dtype):
    """values = flat[kept].copy() and np.zeros(d, values.dtype) keep the input
    dtype in the reference (compressor.py:94,101): integer and float16 inputs
    rank in an exact widening on the device and come back in their own dtype;
    frames carry the same f32 wire values as the reference's astype('<f4')."""
    rng = np.random.default_rng(5)
    if dtype == np.float16:
        x = rng.standard_normal(50_000).astype(np.float16)
    else:  # many exact ties: the lower-index rule decides most of the kept set
        x = rng.integers(-1000, 1000, size=50_000).astype(dtype)
    for ratio in (10.0, 100.0):
        p = P.topk_compress(x, ratio)
        vals, idx, d = O.topk_compress(x, ratio, method="argsort")
        assert p.values.dtype == torch.from_numpy(vals).dtype
        assert np.array_equal(p.indices.cpu().numpy(), idx)
        assert np.array_equal(p.values.cpu().numpy(), vals)
        assert p.to_bytes() == O.to_bytes(vals, idx, d)
        dense = P.topk_decompress(p)
        ref = O.topk_decompress(vals, idx, d)
        assert dense.dtype == torch.from_numpy(ref).dtype
        assert np.array_equal(dense.cpu().numpy(), ref)
        # the same through a CUDA tensor of that dtype, and a modified payload (repacked frame)
        pt = P.topk_compress(torch.from_numpy(x).to(cuda), ratio)
        assert pt.values.dtype == p.values.dtype and torch.equal(pt.indices, p.indices)
        q = dataclasses.replace(pt, values=pt.values.clone())
        assert q.to_bytes() == O.to_bytes(vals, idx, d)
        assert torch.equal(P.topk_decompress(q), dense)


def test_fp64_nan_payload_in_frames(cuda):
    """kept fp64 NaNs reach the f32 wire value as NaN (the payload
    bits may differ from numpy's astype('<f4')); indices and every non-NaN
    value are bit-exact, and the decompressed fp64 vector keeps the input bits."""
    x = np.array([1.5, np.nan, -2.25, 0.0, 3.0, -np.inf, 7.0, np.nan], dtype=np.float64)
    x.view(np.uint64)[1] = 0x7FF8_0000_DEAD_BEEF  # quiet NaN with a payload
    x.view(np.uint64)[7] = 0xFFF4_0000_0000_0001  # negative signalling-pattern NaN
    for ratio in (1.0, 8.0 / 7.0, 2.0):
        p = P.topk_compress(torch.from_numpy(x).to(cuda), ratio)
        vals, idx, d = O.topk_compress(x, ratio, method="argsort")
        assert np.array_equal(p.indices.cpu().numpy(), idx)
        assert np.array_equal(p.values.cpu().numpy().view(np.uint64), vals.view(np.uint64))  # fp64 values: exact
        got = np.frombuffer(p.to_bytes(), dtype="<f4", offset=16 + 8 * len(idx))
        ref = vals.astype("<f4")
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(got), nan)
        assert np.array_equal(got[~nan].view(np.uint32), ref[~nan].view(np.uint32))
        dense = P.topk_decompress(p).cpu().numpy()
        assert np.array_equal(dense.view(np.uint64), O.topk_decompress(vals, idx, d).view(np.uint64))
