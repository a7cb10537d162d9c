"""GPU parity of the sm_100a kernels against the reference (golden frames) and the oracle.

Bar: bit-exact.  Compressed frames must equal the reference's
SparsePayload.to_bytes() byte-for-byte; decompressed tensors must equal the
reference's topk_decompress bit-for-bit.
"""
import ctypes
import itertools

import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import paper_2410_12707_b200 as P
from paper_2410_12707_b200 import _lib
from golden_cases import cases, plans
from oracle import compressor_oracle as O

pytestmark = pytest.mark.gpu


def _bits(t: torch.Tensor) -> np.ndarray:
    a = t.detach().cpu()
    if a.dtype == torch.bfloat16:
        return a.view(torch.int16).numpy().view(np.uint16)
    return a.numpy().view({4: np.uint32, 8: np.uint64}[a.element_size()])


def _bf16_tensor(bits: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).to(device)


# --------------------------------------------------------------------------- golden frames


@pytest.mark.parametrize("prefix", ["f32", "f64"])
def test_golden_frames_bit_exact(cuda, prefix):
    bad = []
    for name, x, ratio, frame in cases(prefix):
        p = P.topk_compress(torch.from_numpy(x.copy()).to(cuda), ratio)
        if p.to_bytes() != frame:
            bad.append(name)
    assert not bad, f"{len(bad)} frames differ, e.g. {bad[:10]}"


def test_golden_frames_bf16(cuda):
    for name, bits, ratio, frame in cases("bf16"):
        x = _bf16_tensor(bits, cuda)
        p = P.topk_compress(x, ratio)
        assert p.to_bytes() == frame, name
        assert p.values.dtype == torch.bfloat16
        # values (dtype preserved) agree with the frame's f32 values exactly
        _, idx, d = O.from_bytes(frame)
        np.testing.assert_array_equal(_bits(p.values), bits[idx])


def test_golden_decompress_bit_exact(cuda):
    for name, x, ratio, frame in itertools.islice(cases("f32"), 0, None, 7):
        p = P.topk_compress(torch.from_numpy(x.copy()).to(cuda), ratio)
        dense = P.topk_decompress(p)
        vals, idx, d = O.topk_compress(x, ratio)
        ref = O.topk_decompress(vals, idx, d)
        assert dense.dtype == torch.float32
        np.testing.assert_array_equal(_bits(dense), ref.view(np.uint32), err_msg=name)


def test_from_bytes_round_trip(cuda):
    for name, x, ratio, frame in itertools.islice(cases("f32"), 0, None, 13):
        q = P.SparsePayload.from_bytes(frame, device=cuda)
        assert q.values.dtype == torch.float64 and q.to_bytes() == frame
        dense = P.topk_decompress(q)
        vals, idx, d = O.from_bytes(frame)
        np.testing.assert_array_equal(dense.cpu().numpy(), O.topk_decompress(vals, idx, d), err_msg=name)


# --------------------------------------------------------------------------- reference unit tests, on the GPU


class TestReferenceUnitTests:
    """The reference's tests/test_compressor.py:33-118, run against the GPU path."""

    def test_two_largest(self, cuda):
        p = P.topk_compress([0.1, -5.0, 3.0, 0.0], 2)
        assert p.indices.tolist() == [1, 2]
        assert p.values.tolist() == [-5.0, 3.0]

    def test_ratio_one_identity(self, cuda):
        v = [1.0, -2.0, 0.5]
        p = P.topk_compress(v, 1)
        assert p.k == 3
        assert P.topk_decompress(p).tolist() == v

    def test_magnitude_tie_lower_index(self, cuda):
        p = P.topk_compress([2.0, -2.0, 1.0], 3)
        assert p.indices.tolist() == [0] and p.values.tolist() == [2.0]

    def test_empty_vector(self, cuda):
        with pytest.raises(P.EmptyVector):
            P.topk_compress([], 2)
        with pytest.raises(P.EmptyVector):
            P.topk_compress(torch.empty(0, device=cuda), 2)

    def test_dtype_preserved(self, cuda):
        p = P.topk_compress(np.array([1.0, 2.0], dtype=np.float64), 2)
        assert p.values.dtype == torch.float64

    @settings(max_examples=200, deadline=None)
    @given(st.lists(st.floats(-100, 100), min_size=1, max_size=12), st.floats(1, 20))
    def test_matches_brute_force(self, cuda, values, ratio):
        p = P.topk_compress(values, ratio)
        k = P.select_k(len(values), ratio)
        best = None
        for combo in itertools.combinations(range(len(values)), k):
            score = tuple(sorted((abs(values[i]) for i in combo), reverse=True))
            if best is None or score > best[0]:
                best = (score, combo)
        assert set(p.indices.tolist()) == set(best[1])

    @settings(max_examples=50, deadline=None)
    @given(st.lists(st.floats(-100, 100), min_size=2, max_size=30))
    def test_error_monotone_in_kept_count(self, cuda, values):
        v = torch.tensor(values, dtype=torch.float64, device=cuda)
        errs = []
        for ratio in (8, 4, 2, 1):
            rec = P.topk_decompress(P.topk_compress(v, ratio))
            errs.append(float(torch.linalg.norm(v - rec)))
        assert all(a >= b - 1e-12 for a, b in zip(errs, errs[1:]))

    def test_inverse_on_support(self, cuda):
        p = P.topk_compress([0.1, -5.0, 3.0, 0.0], 2)
        assert P.topk_decompress(p).tolist() == [0.0, -5.0, 3.0, 0.0]

    def test_all_zero_vector(self, cuda):
        assert P.topk_decompress(P.topk_compress(np.zeros(8), 4)).tolist() == [0.0] * 8

    def test_payload_matches_wire_bytes(self, cuda):
        rng = np.random.default_rng(1)
        for d, ratio in [(10, 2), (100, 100), (7, 3.5)]:
            p = P.topk_compress(rng.standard_normal(d), ratio)
            assert p.payload_nbytes == P.wire_bytes(d, ratio)
            assert len(p.to_bytes()) == 16 + P.wire_bytes(d, ratio)

    def test_byte_round_trip(self, cuda):
        p = P.topk_compress(np.array([1.5, -2.25, 0.125, 4.0], dtype=np.float32), 2)
        q = P.SparsePayload.from_bytes(p.to_bytes())
        assert q.original_len == 4 and q.indices.tolist() == p.indices.tolist()
        assert q.values.tolist() == p.values.tolist()


# --------------------------------------------------------------------------- sizes of the BASELINE configs


def _check_against_oracle(x: torch.Tensor, ratio: float):
    p = P.topk_compress(x, ratio)
    xf = x.float() if x.dtype == torch.bfloat16 else x
    host = xf.cpu().numpy()
    vals, idx, d = O.topk_compress(host, ratio, method="threshold")
    got_idx = p.indices.cpu().numpy()
    np.testing.assert_array_equal(got_idx, idx)
    assert p.to_bytes() == O.to_bytes(vals, idx, d)
    return p


@pytest.mark.parametrize("ratio", [10, 100, 1000, 10000])
def test_c1_gpt2_small_activation(cuda, ratio):
    """configs[0]: 8x1024x768 fp32 (d = 6,291,456)."""
    g = torch.Generator(device=cuda).manual_seed(0)
    x = torch.randn(8, 1024, 768, device=cuda, generator=g)
    p = _check_against_oracle(x, ratio)
    dense = P.topk_decompress(p)
    ref = torch.zeros_like(x.reshape(-1))
    ref[p.indices] = x.reshape(-1)[p.indices]
    assert torch.equal(dense.view(torch.int32), ref.view(torch.int32))


@pytest.mark.parametrize("dist", ["relu", "laplace", "student_t", "outlier_channels", "quantized"])
def test_c1_variants(cuda, dist):
    g = torch.Generator(device=cuda).manual_seed(1)
    x = torch.randn(8, 1024, 768, device=cuda, generator=g)
    if dist == "relu":
        x = torch.relu(x)
        ratios = (1.5, 10, 100)
    elif dist == "laplace":
        x = torch.sign(x) * torch.log1p(x.abs() * 10)
        ratios = (100,)
    elif dist == "student_t":
        x = x / torch.sqrt((torch.randn(x.shape, device=cuda, generator=g) ** 2 +
                            torch.randn(x.shape, device=cuda, generator=g) ** 2 +
                            torch.randn(x.shape, device=cuda, generator=g) ** 2) / 3)
        ratios = (10, 1000)
    elif dist == "outlier_channels":
        x[..., ::97] *= 50.0  # GPT-2 style massive-activation channels
        ratios = (100, 1000)
    else:
        x = torch.round(x * 2) / 2
        ratios = (10, 100)
    for r in ratios:
        _check_against_oracle(x.contiguous(), r)


@pytest.mark.parametrize("shape", [(64, 2048, 7, 7), (64, 1024, 14, 14), (64, 512, 28, 28)])
def test_resnet101_boundaries_vs_oracle(cuda, shape):
    g = torch.Generator(device=cuda).manual_seed(2)
    act = torch.relu(torch.randn(shape, device=cuda, generator=g))
    grad = torch.randn(shape, device=cuda, generator=g) * 1e-3
    for r in (10, 100, 1000):
        _check_against_oracle(act, r)
        _check_against_oracle(grad, r)


def test_resnet101_largest_boundary_properties(cuda):
    """[64,256,56,56] (d = 51,380,224): size-independent properties, no CPU sort."""
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.relu(torch.randn(64, 256, 56, 56, device=cuda, generator=g)).reshape(-1)
    for r in (10, 100, 1000):
        p = P.topk_compress(x, r)
        k = P.select_k(x.numel(), r)
        idx = p.indices
        assert idx.numel() == k
        assert bool((idx[1:] > idx[:-1]).all())
        assert torch.equal(p.values, x[idx])
        kept = torch.zeros(x.numel(), dtype=torch.bool, device=cuda)
        kept[idx] = True
        a = x.abs()
        t_min = a[kept].min()
        assert bool((a[~kept] <= t_min).all())
        # ties at the threshold: every dropped element equal to the threshold lies after every kept one
        eq_dropped = torch.nonzero((~kept) & (a == t_min)).reshape(-1)
        eq_kept = torch.nonzero(kept & (a == t_min)).reshape(-1)
        if eq_dropped.numel() and eq_kept.numel():
            assert int(eq_dropped.min()) > int(eq_kept.max())
        dense = P.topk_decompress(p)
        assert torch.equal(dense[idx], x[idx]) and int(torch.count_nonzero(dense[~kept])) == 0


def test_bf16_large_vs_oracle(cuda):
    g = torch.Generator(device=cuda).manual_seed(4)
    x = torch.randn(8, 1024, 1024, device=cuda, generator=g).to(torch.bfloat16)
    for r in (10, 100):
        p = _check_against_oracle(x, r)
        assert torch.equal(p.values, x.reshape(-1)[p.indices])
        dense = P.topk_decompress(p)
        assert dense.dtype == torch.bfloat16


def test_bf16_heavy_ties_vs_oracle(cuda):
    """bf16 at 16M elements, r=10 and 3: tens of thousands of keys equal the
    threshold value (bf16 has 128 values per octave), far beyond the
    final-candidate window capacity; ties must still go to the lower indices."""
    g = torch.Generator(device=cuda).manual_seed(44)
    x = torch.randn(16 * 1024 * 1024, device=cuda, generator=g).to(torch.bfloat16)
    for r in (10, 3):
        p = _check_against_oracle(x, r)
        assert torch.equal(p.values, x.reshape(-1)[p.indices])


def test_f64_vs_oracle(cuda):
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.randn(300_001, device=cuda, generator=g, dtype=torch.float64)
    for r in (3, 100):
        _check_against_oracle(x, r)


@pytest.mark.parametrize("d", [1, 2, 3, 7, 8, 9, 31, 33, 255, 4097, 16385, 100_001, 1_000_003])
def test_odd_sizes(cuda, d):
    g = torch.Generator(device=cuda).manual_seed(d)
    x = torch.randn(d, device=cuda, generator=g)
    for r in (1, 1.7, 10, 1000):
        _check_against_oracle(x, r)


def test_unaligned_input(cuda):
    g = torch.Generator(device=cuda).manual_seed(6)
    base = torch.randn(100_003, device=cuda, generator=g)
    for off in (1, 2, 3):
        _check_against_oracle(base[off:], 50)


def test_deterministic_repeat(cuda):
    g = torch.Generator(device=cuda).manual_seed(7)
    x = torch.randn(4, 1024, 1600, device=cuda, generator=g)
    frames = {P.topk_compress(x, 300).to_bytes() for _ in range(5)}
    assert len(frames) == 1


def test_workspace_reuse_across_sizes_and_dtypes(cuda):
    """The workspace is left clean by every call (zeroed once)."""
    g = torch.Generator(device=cuda).manual_seed(8)
    xs = [torch.randn(n, device=cuda, generator=g) for n in (1000, 3_000_000, 17, 250_000)]
    for _ in range(2):
        for x in xs:
            _check_against_oracle(x, 37)
            _check_against_oracle(x.to(torch.bfloat16), 11)


def test_side_stream(cuda):
    s = torch.cuda.Stream()
    g = torch.Generator(device=cuda).manual_seed(9)
    x = torch.randn(2_000_000, device=cuda, generator=g)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        p = P.topk_compress(x, 100)
        dense = P.topk_decompress(p)
    s.synchronize()
    vals, idx, d = O.topk_compress(x.cpu().numpy(), 100, method="threshold")
    np.testing.assert_array_equal(p.indices.cpu().numpy(), idx)
    assert torch.equal(dense.cpu()[idx], x.cpu()[idx])


# --------------------------------------------------------------------------- decompress edge cases


def test_decompress_out_of_range(cuda):
    for idx in ([0, 5], [-1, 2], [3]):
        p = P.SparsePayload(values=torch.ones(len(idx), device=cuda),
                            indices=torch.tensor(idx, device=cuda, dtype=torch.int64), original_len=3)
        with pytest.raises(P.IndexOutOfRange):
            P.topk_decompress(p)


def test_decompress_unsorted_and_repeated_last_write_wins(cuda):
    rng = np.random.default_rng(11)
    d = 100_000
    idx = rng.integers(0, d, 20_000)
    vals = rng.standard_normal(20_000).astype(np.float32)
    ref = np.zeros(d, np.float32)
    ref[idx] = vals
    p = P.SparsePayload(values=torch.from_numpy(vals).to(cuda), indices=torch.from_numpy(idx).to(cuda),
                        original_len=d)
    out = P.topk_decompress(p)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)


def test_decompress_accumulate_residual(cuda):
    g = torch.Generator(device=cuda).manual_seed(12)
    x = torch.randn(1_000_000, device=cuda, generator=g)
    base = torch.randn(1_000_000, device=cuda, generator=g)
    p = P.topk_compress(x, 100)
    out = base.clone()
    P.topk_decompress(p, out=out, accumulate=True)
    ref = base.clone()
    ref[p.indices] += x[p.indices]
    assert torch.equal(out, ref)


def test_decompress_k_zero_and_int32_indices(cuda):
    p = P.SparsePayload(values=torch.empty(0, device=cuda), indices=torch.empty(0, dtype=torch.int64, device=cuda),
                        original_len=10)
    assert P.topk_decompress(p).tolist() == [0.0] * 10
    x = torch.randn(50_000, device=cuda)
    q = P.topk_compress(x, 10)
    q32 = P.SparsePayload(values=q.values, indices=q.indices.to(torch.int32), original_len=q.original_len)
    assert torch.equal(P.topk_decompress(q32), P.topk_decompress(q))


# --------------------------------------------------------------------------- C-ABI directly


def test_cabi_frame_entry_points(cuda):
    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(13)
    x = torch.randn(1_234_567, device=cuda, generator=g)
    d, r = x.numel(), 77.0
    k = P.select_k(d, r)
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda)
    wsb = L.gp_topk_workspace_bytes(d, _lib.DTYPE_F32)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    assert L.gp_workspace_init(ws.data_ptr(), wsb, s) == 0
    assert L.gp_topk_compress_frame(x.data_ptr(), _lib.DTYPE_F32, d, k, frame.data_ptr(), ws.data_ptr(), wsb, s) == 0
    assert frame.cpu().numpy().tobytes() == O.compress_frame(x.cpu().numpy(), r, "threshold")
    out = torch.empty(d, device=cuda)
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), _lib.DTYPE_F32, 0, err.data_ptr(), s) == 0
    assert int(err.item()) == 0
    vals, idx, _ = O.from_bytes(frame.cpu().numpy().tobytes())
    np.testing.assert_array_equal(out.cpu().numpy(), O.topk_decompress(vals.astype(np.float32), idx, d))
    # int32 index output
    i32 = torch.empty(k, dtype=torch.int32, device=cuda)
    v32 = torch.empty(k, device=cuda)
    assert L.gp_topk_compress(x.data_ptr(), 0, d, k, i32.data_ptr(), 4, v32.data_ptr(), 0, None, None,
                              ws.data_ptr(), wsb, s) == 0
    np.testing.assert_array_equal(i32.cpu().numpy(), idx)
    # argument validation
    assert L.gp_topk_compress(x.data_ptr(), 0, 0, 1, i32.data_ptr(), 4, v32.data_ptr(), 0, None, None,
                              ws.data_ptr(), wsb, s) == 2
    assert L.gp_topk_compress(x.data_ptr(), 0, d, d + 1, i32.data_ptr(), 4, v32.data_ptr(), 0, None, None,
                              ws.data_ptr(), wsb, s) == 6


def test_device_plan_matches_reference(cuda):
    for R, r, expected in plans():
        Rt = torch.tensor(R, dtype=torch.float64, device=cuda)
        dl = torch.full((len(R),), 6291456, dtype=torch.int64, device=cuda)
        rr, kk, stt = P.adatopk_plan_device(Rt, r, dl)
        assert int(stt.item()) == 0
        assert rr.cpu().tolist() == expected
        assert kk.cpu().tolist() == [O.select_k(6291456, e) for e in expected]
    _, _, stt = P.adatopk_plan_device(torch.zeros(2, dtype=torch.float64, device=cuda), 10,
                                      torch.ones(2, dtype=torch.int64, device=cuda))
    assert int(stt.item()) == 4  # NoCommunication


def test_host_pinned_input_e2e(cuda):
    x = torch.randn(3_000_000).pin_memory()
    p = P.topk_compress(x, 100)
    vals, idx, d = O.topk_compress(x.numpy(), 100, method="threshold")
    np.testing.assert_array_equal(p.indices.cpu().numpy(), idx)


@pytest.mark.parametrize("ratio", [3, 10, 30, 100, 1000, 20000])
def test_decompress_frame_large_k_both_kernels(cuda, ratio):
    """Both fast decompress kernels (tiled, dense payloads; fill+scatter, sparse
    payloads) at k large enough that the probe bracket is wider than one entry:
    no spurious error flag, and the output equals x on the support, 0 elsewhere."""
    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(ratio)
    x = torch.randn(12_845_056, device=cuda, generator=g)
    d = x.numel()
    k = P.select_k(d, ratio)
    s = torch.cuda.current_stream().cuda_stream
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda)
    wsb = L.gp_topk_workspace_bytes(d, _lib.DTYPE_F32)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda)
    assert L.gp_workspace_init(ws.data_ptr(), wsb, s) == 0
    assert L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, s) == 0
    out = torch.full((d,), float("nan"), device=cuda)
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(), s) == 0
    assert int(err.item()) == 0
    idx = frame[16:16 + 8 * k].view(torch.int64)
    ref = torch.zeros_like(x)
    ref[idx] = x[idx]
    assert torch.equal(out, ref)


@pytest.mark.parametrize("ratio", [10, 1000])
def test_capped_grid_and_concurrent_streams_identical_frames(cuda, ratio):
    """gp_topk_compress_frame_ctas: any grid cap (1 CTA .. one per SM) gives the
    byte-identical reference frame, also with four compresses in flight on
    four streams (one workspace each), as the benchmark runs them."""
    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(ratio)
    xs = [torch.relu(torch.randn(2_000_003, device=cuda, generator=g)) if i % 2 else
          torch.randn(2_000_003, device=cuda, generator=g) * 1e-3 for i in range(4)]
    d = xs[0].numel()
    k = P.select_k(d, ratio)
    wsb = L.gp_topk_workspace_bytes(d, _lib.DTYPE_F32)
    wss = [torch.zeros(wsb, dtype=torch.uint8, device=cuda) for _ in range(4)]
    expect = [O.compress_frame(x.cpu().numpy(), ratio, "threshold") for x in xs]
    s = torch.cuda.current_stream().cuda_stream
    for ctas in (1, 7, 37, 74, 0):
        f = torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda)
        assert L.gp_topk_compress_frame_ctas(xs[0].data_ptr(), 0, d, k, f.data_ptr(), wss[0].data_ptr(), wsb, s,
                                             ctas) == 0
        assert f.cpu().numpy().tobytes() == expect[0], ctas
    streams = [torch.cuda.Stream(cuda) for _ in range(4)]
    frames = [torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda) for _ in range(4)]
    torch.cuda.synchronize()
    for rep in range(3):
        for i, st in enumerate(streams):
            assert L.gp_topk_compress_frame_ctas(xs[i].data_ptr(), 0, d, k, frames[i].data_ptr(), wss[i].data_ptr(),
                                                 wsb, st.cuda_stream, 37) == 0
        torch.cuda.synchronize()
        for i in range(4):
            assert frames[i].cpu().numpy().tobytes() == expect[i], (rep, i)


@pytest.mark.parametrize("layout", ["spread", "clustered"])
def test_many_final_candidates(cuda, layout):
    """40,000 distinct values inside one fine histogram bin, with the k-th
    largest among them.  'spread': every CTA holds a few hundred of them (the
    fast path, extras read from the CTA regions).  'clustered': one CTA's
    range holds them all and overflows its region (every CTA falls back to the
    slow path after B2).  Both must equal the reference selection."""
    d, hot = 2_500_000, 40_000
    g = torch.Generator(device=cuda).manual_seed(17)
    x = torch.rand(d, device=cuda, generator=g) * 0.5
    vals = 1.0 + torch.rand(hot, device=cuda, generator=g) * 2.0 ** -10
    pos = (torch.arange(hot, device=cuda) * (d // hot) if layout == "spread"
           else torch.arange(hot, device=cuda) + 100_000)
    x[pos] = vals
    ratio = d / 20_000
    _check_against_oracle(x, ratio)


def _decompress_flags(cuda, idx, vals, d, cases, mode=0):
    """Run the fast decompress once per case (each case mutates `idx` in place,
    launches, and undoes the mutation, all stream-ordered) and return the
    validation flag of every launch."""
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    out = torch.zeros(d, device=cuda)
    err = torch.zeros(len(cases) + 1, dtype=torch.int32, device=cuda)
    k = idx.numel()

    def launch(slot):
        assert L.gp_topk_decompress(idx.data_ptr(), 8, vals.data_ptr(), 0, k, d, out.data_ptr(), 0, mode,
                                    err[slot:].data_ptr(), s) == 0

    launch(0)
    for c, (kind, j) in enumerate(cases, 1):
        saved = idx[j:j + 2].clone()
        if kind == "swap":
            idx[j:j + 2] = saved.flip(0)
        else:  # "dup": idx[j+1] = idx[j]
            idx[j + 1:j + 2] = saved[:1]
        launch(c)
        idx[j:j + 2] = saved
    return err.cpu().numpy()


def _sorted_unique(rng, lo, hi, n):
    return np.sort(rng.choice(np.arange(lo, hi, dtype=np.int64), n, replace=False))


@pytest.mark.parametrize("layout", ["uniform", "uniform_accumulate", "clustered", "large", "sparse"])
def test_decompress_sortedness_flag_is_exact(cuda, layout):
    """The fast decompress kernels validate strict increase in the same launch
    (each CTA checks its share of the adjacent pairs).  No false positive on
    sorted input (it would cost a general re-run), and every single violation
    is flagged: one adjacent swap or duplicate, placed next to every
    4096-aligned output position (every possible CTA boundary, where a CTA's
    entries start) and at random.  Tiled kernel for all layouts but 'sparse'
    (fill + scatter)."""
    rng = np.random.default_rng(23)
    if layout.startswith("uniform"):
        d = 4 << 20
        h = _sorted_unique(rng, 0, d, d // 10)
    elif layout == "clustered":  # two dense clusters, long empty stretches (probe window misses)
        d = 4 << 20
        h = np.concatenate([_sorted_unique(rng, 100_000, 400_000, 150_000),
                            _sorted_unique(rng, 3_000_000, 3_200_000, 150_000)])
    elif layout == "large":  # > 64 MB output: tiled kernel at r = 100
        d = 20 << 20
        h = _sorted_unique(rng, 0, d, d // 100)
    else:  # k/d = 1/100, 16 MB output: fill + scatter kernel
        d = 4 << 20
        h = _sorted_unique(rng, 0, d, d // 100)
    k = h.size
    step = 4096 if d <= (4 << 20) else 9 * 4096
    lbs = np.searchsorted(h, np.arange(step, d, step))
    pos = set()
    for lb in lbs:
        pos.update((int(lb) - 2, int(lb) - 1, int(lb)))
    pos.update(int(p) for p in rng.integers(0, k - 1, 200))
    pos.update((0, 1, 510, 511, 512, k - 3, k - 2))
    pos = sorted(p for p in pos if 0 <= p <= k - 2)
    cases = [("swap", p) for p in pos] + [("dup", int(p)) for p in rng.choice(pos, 100, replace=False)]
    idx = torch.from_numpy(h).to(cuda)
    vals = torch.randn(k, device=cuda)
    flags = _decompress_flags(cuda, idx, vals, d, cases, mode=1 if layout.endswith("accumulate") else 0)
    assert flags[0] == 0, "false positive on sorted input"
    missed = [c for c, f in zip(cases, flags[1:]) if not f & _lib.FLAG_UNSORTED]
    assert not missed, missed[:10]
    np.testing.assert_array_equal(idx.cpu().numpy(), h)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_maximum_vector_length(cuda, dtype):
    """d = 2^31 - 1 (8.6 GB of fp32, the kernels' index width) compresses and
    round-trips, checked by size-independent properties: k strictly increasing
    indices, every kept |x| >= every dropped |x| with magnitude ties resolved to
    the lowest indices, decompress = x on the support and 0 elsewhere.
    d = 2^31 is rejected with an argument error rather than truncated.  fp32
    and bf16 (selection on the exact fp32 upcast)."""
    n = 1 << 31
    g = torch.Generator(device=cuda).manual_seed(31)
    buf = torch.empty(n, device=cuda, dtype=dtype)
    buf.normal_(generator=g)  # bf16: ~32K distinct magnitudes, so the tie rule decides most of the selection
    x = buf[: n - 1]
    d, ratio = x.numel(), 1e4
    p = P.topk_compress(x, ratio)
    k = P.select_k(d, ratio)
    idx = p.indices
    assert idx.numel() == k and bool((idx[1:] > idx[:-1]).all()) and int(idx[0]) >= 0 and int(idx[-1]) < d
    kept = x[idx].float().abs()
    thr = float(kept.min())
    a = x.float().abs()
    a[idx] = -1.0
    assert float(a.max()) <= thr
    tied_dropped = torch.nonzero(a == thr).flatten()
    if tied_dropped.numel():
        assert int(idx[kept == thr].max()) < int(tied_dropped.min())
    del a, tied_dropped
    out = P.topk_decompress(p)
    assert torch.equal(out[idx], x[idx])
    out[idx] = 0.0
    assert int(torch.count_nonzero(out)) == 0
    del out, p
    torch.cuda.empty_cache()
    with pytest.raises(ValueError):
        P.topk_compress(buf, ratio)


def test_decompress_skips_sync_only_for_unmodified_payloads(cuda):
    """A payload made by topk_compress decompresses without reading the
    validation flag back; replacing or modifying its indices (or its length)
    restores the reference's synchronous IndexOutOfRange check."""
    import dataclasses

    x = torch.randn(100_000, device=cuda)
    p = P.topk_compress(x, 10)
    ref = torch.zeros_like(x)
    ref[p.indices] = x[p.indices]
    assert torch.equal(P.topk_decompress(p), ref)
    q = P.topk_compress(x, 10)
    q.indices[0] = -1  # in place (a view of the frame): the version changes
    with pytest.raises(P.IndexOutOfRange):
        P.topk_decompress(q)
    r = P.topk_compress(x, 10)
    bad = r.indices.clone()
    bad[-1] = 10 ** 6
    with pytest.raises(P.IndexOutOfRange):
        P.topk_decompress(dataclasses.replace(r, indices=bad))
    s = P.topk_compress(x, 10)
    s.original_len = 50_000
    with pytest.raises(P.IndexOutOfRange):
        P.topk_decompress(s)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float64])
def test_decompress_accumulate_bf16_f64(cuda, dtype):
    """Residual mode (tiled kernel) in bf16 and f64: out[idx] += vals, rounded
    like torch (bf16: fp32 add, round to nearest even), bit for bit."""
    g = torch.Generator(device=cuda).manual_seed(21)
    x = torch.randn(3_000_000, device=cuda, generator=g).to(dtype)
    base = torch.randn(3_000_000, device=cuda, generator=g).to(dtype)
    p = P.topk_compress(x, 50)
    out = base.clone()
    P.topk_decompress(p, out=out, accumulate=True)
    ref = base.clone()
    ref[p.indices] += x[p.indices]
    assert torch.equal(out.view(torch.int16 if dtype == torch.bfloat16 else torch.int64),
                       ref.view(torch.int16 if dtype == torch.bfloat16 else torch.int64))


@pytest.mark.parametrize("ratio", [10, 100])
def test_decompress_frame_misaligned_output(cuda, ratio):
    """An output pointer that is not 16-byte aligned takes the element-wise store
    path (bulk TMA stores need 16-byte alignment); the result is still exact."""
    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(ratio)
    x = torch.randn(2_000_000, device=cuda, generator=g)
    d = x.numel()
    p = P.topk_compress(x, ratio)
    k = p.k
    buf = torch.full((d + 1,), float("nan"), device=cuda)
    out = buf[1:]  # 4-byte offset
    assert out.data_ptr() % 16 != 0
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    assert L.gp_topk_decompress_frame(p.frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(), s) == 0
    assert int(err.item()) == 0
    ref = torch.zeros_like(x)
    ref[p.indices] = x[p.indices]
    assert torch.equal(out, ref) and bool(torch.isnan(buf[0]))


def test_tensor_on_another_device_than_current(cuda):
    """A tensor on cuda:1 while cuda:0 is current: the drop-in launches on the
    tensor's GPU and the frame equals the one produced on cuda:0."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run under gpurun --gpus 2)")
    g = torch.Generator(device=cuda).manual_seed(5)
    x0 = torch.randn(1_500_000, device=cuda, generator=g)
    x1 = x0.to("cuda:1")
    with torch.cuda.device(0):
        p1 = P.topk_compress(x1, 100)
        d1 = P.topk_decompress(p1)
    p0 = P.topk_compress(x0, 100)
    assert p1.indices.device.index == 1 and d1.device.index == 1
    assert p1.to_bytes() == p0.to_bytes()
    assert torch.equal(d1.cpu(), P.topk_decompress(p0).cpu())
