"""GPU parity of the single-cluster compress (csrc/gp_cluster.cu) for short vectors.

Vectors up to one 8-CTA cluster's shared memory (393,216 fp32 / 786,432 bf16
/ 196,608 fp64 elements) can go through the cluster kernel instead of the
cooperative grid (by default those of at most 98,304 elements).  Bar: frames bit-exact against the oracle (itself pinned to
frames made by the reference, tests/test_oracle_golden.py), and identical to
the cooperative kernel's frames on the same input (gp_set_cluster_path(0)).
"""
import numpy as np
import pytest
import torch

import paper_2410_12707_b200 as P
from paper_2410_12707_b200 import _lib
from paper_2410_12707_b200.transport import FrameCodec
from oracle import compressor_oracle as O

pytestmark = pytest.mark.gpu

CAP_F32, CAP_BF16, CAP_F64 = 393_216, 786_432, 196_608


def _host(x: torch.Tensor) -> np.ndarray:
    return (x.float() if x.dtype == torch.bfloat16 else x).cpu().numpy().reshape(-1)


def _frame(x: torch.Tensor, ratio: float) -> bytes:
    p = P.topk_compress(x, ratio)
    torch.cuda.synchronize()
    return p.to_bytes()


class _Path:
    """Route compresses through the cluster kernel wherever the vector fits it
    (True: gp_set_cluster_path mode 2) or through the cooperative grid (False: mode 0)."""

    def __init__(self, cluster: bool):
        self.cluster = cluster

    def __enter__(self):
        self.prev = _lib.lib().gp_set_cluster_path(2 if self.cluster else 0)

    def __exit__(self, *exc):
        _lib.lib().gp_set_cluster_path(self.prev)


def _check(x: torch.Tensor, ratio: float, both_paths: bool = True):
    ref = O.compress_frame(_host(x), ratio, method="threshold")
    with _Path(True):
        got = _frame(x, ratio)
    assert got == ref, f"cluster path frame differs (d={x.numel()}, r={ratio}, {x.dtype})"
    if both_paths:
        with _Path(False):
            assert _frame(x, ratio) == ref, f"cooperative path frame differs (d={x.numel()}, r={ratio})"


@pytest.mark.parametrize("d", [1, 2, 3, 7, 15, 16, 17, 31, 1000, 4095, 4097, 65_537, 262_147, CAP_F32])
@pytest.mark.parametrize("ratio", [1.5, 10.0, 100.0, 1e4])
def test_cluster_fp32_sizes(cuda, d, ratio):
    g = torch.Generator(device=cuda).manual_seed(d * 7 + int(ratio))
    _check(torch.randn(d, device=cuda, generator=g), ratio, both_paths=d >= 1000)


def test_cluster_capacity_boundary(cuda):
    """One element past the cluster's capacity goes to the cooperative grid; both bit-exact."""
    g = torch.Generator(device=cuda).manual_seed(5)
    for d in (CAP_F32 - 1, CAP_F32, CAP_F32 + 1):
        _check(torch.randn(d, device=cuda, generator=g), 100.0, both_paths=False)


def _special(d: int, kind: str, cuda) -> torch.Tensor:
    g = torch.Generator(device=cuda).manual_seed(11)
    x = torch.randn(d, device=cuda, generator=g)
    if kind == "all_equal":
        return torch.full((d,), 0.5, device=cuda)
    if kind == "ties_small_range":  # integers in [-3, 3]: huge tie groups at the threshold
        return torch.randint(-3, 4, (d,), device=cuda, generator=g).float()
    if kind == "nan_inf_zero":
        x[::7] = float("nan")
        x[1::11] = float("inf")
        x[2::13] = -float("inf")
        x[3::5] = 0.0
        x[4::9] = -0.0
        x[5::17] = 1e-42  # denormal
        return x
    if kind == "all_nan":
        return torch.full((d,), float("nan"), device=cuda)
    if kind == "ascending":
        return torch.arange(d, device=cuda, dtype=torch.float32)
    if kind == "descending":
        return -torch.arange(d, device=cuda, dtype=torch.float32)
    if kind == "relu":
        return torch.relu(x)
    if kind == "half_equal":  # the first CTAs' top bins overflow their lists, the last ones' do not
        x[: d // 2] = 0.75
        return x
    if kind == "neg_nan_payloads":
        v = x.view(torch.int32)
        v[::3] = torch.tensor(-4194305, dtype=torch.int32, device=cuda)  # 0xFFBFFFFF: a -NaN with payload
        return x
    raise ValueError(kind)


KINDS = ["all_equal", "ties_small_range", "nan_inf_zero", "all_nan", "ascending", "descending", "relu",
         "neg_nan_payloads", "half_equal"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("ratio", [2.0, 10.0, 1000.0])
def test_cluster_distributions(cuda, kind, ratio):
    _check(_special(300_001, kind, cuda), ratio)


@pytest.mark.parametrize("d", [1000, 699_999, CAP_BF16])
@pytest.mark.parametrize("ratio", [10.0, 100.0])
def test_cluster_bf16(cuda, d, ratio):
    g = torch.Generator(device=cuda).manual_seed(d)
    _check(torch.randn(d, device=cuda, generator=g).bfloat16(), ratio)


def test_cluster_bf16_ties(cuda):
    g = torch.Generator(device=cuda).manual_seed(3)
    _check((torch.randint(-8, 9, (500_000,), device=cuda, generator=g).float() / 4).bfloat16(), 7.0)


@pytest.mark.parametrize("d", [1000, CAP_F64])
@pytest.mark.parametrize("ratio", [10.0, 100.0])
def test_cluster_fp64(cuda, d, ratio):
    g = torch.Generator(device=cuda).manual_seed(d + 1)
    x = torch.randn(d, device=cuda, generator=g, dtype=torch.float64)
    x[::101] = float("inf")
    x[7::211] = 0.0
    _check(x, ratio)


@pytest.mark.parametrize("off", [1, 2, 3])
def test_cluster_unaligned_input(cuda, off):
    """A storage offset that breaks 16-byte alignment: the slice is loaded element-wise."""
    g = torch.Generator(device=cuda).manual_seed(off)
    base = torch.randn(200_003 + off, device=cuda, generator=g)
    x = base[off:]
    assert x.data_ptr() % 16 != 0
    _check(x, 10.0)


def test_cluster_decompress_round_trip(cuda):
    g = torch.Generator(device=cuda).manual_seed(8)
    x = torch.randn(8, 1024, 96, device=cuda, generator=g)
    with _Path(True):
        p = P.topk_compress(x, 100.0)
        dense = P.topk_decompress(p)
    vals, idx, d = O.from_bytes(O.compress_frame(_host(x), 100.0, method="threshold"))
    ref = O.topk_decompress(vals.astype(np.float32), idx, d)
    assert np.array_equal(dense.cpu().numpy().reshape(-1).view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("max_ctas", [1, 2, 3, 8, 16])
def test_cluster_capped_grid(cuda, max_ctas):
    """(mode 2) gp_topk_compress_frame_ctas: the cluster never exceeds max_ctas CTAs; a
    vector longer than max_ctas slices goes to the cooperative grid."""
    L = _lib.lib()
    prev = L.gp_set_cluster_path(2)
    for d in (50_000, 200_000, 390_000):
        g = torch.Generator(device=cuda).manual_seed(d + max_ctas)
        x = torch.randn(d, device=cuda, generator=g)
        k = O.select_k(d, 30.0)
        frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=cuda)
        wsb = L.gp_topk_workspace_bytes(d, 0)
        ws = torch.zeros(wsb, dtype=torch.uint8, device=cuda)
        assert L.gp_workspace_init(ws.data_ptr(), wsb, None) == 0
        s = torch.cuda.current_stream().cuda_stream
        assert L.gp_topk_compress_frame_ctas(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, s,
                                             max_ctas) == 0
        torch.cuda.synchronize()
        assert bytes(frame.cpu().numpy()) == O.compress_frame(_host(x), 30.0, method="threshold"), (d, max_ctas)
    L.gp_set_cluster_path(prev)


def test_cluster_device_resident_k(cuda):
    """k read from device memory (on-device AdaTopK plans) on the cluster path,
    including an invalid k, which flags GP_FLAG_BAD_K and writes an invalid header."""
    codec = FrameCodec(cuda)
    prev = _lib.lib().gp_set_cluster_path(2)
    g = torch.Generator(device=cuda).manual_seed(21)
    d = 300_000
    x = torch.randn(d, device=cuda, generator=g)
    for k in (1, 17, 3000, d // 3, d):
        kd = torch.tensor([k], dtype=torch.int64, device=cuda)
        f = codec.compress_dk(x, kd, d)
        torch.cuda.synchronize()
        raw = bytes(f[: 16 + 12 * k].cpu().numpy())
        host = _host(x)
        kept = np.sort(O.topk_indices_threshold(host, k))
        assert raw == O.to_bytes(host[kept], kept, d), k
    codec.check()
    kd = torch.tensor([d + 5], dtype=torch.int64, device=cuda)
    codec.compress_dk(x, kd, d)
    with pytest.raises(ValueError):
        codec.check()
    _lib.lib().gp_set_cluster_path(prev)


def test_cluster_repeatable_and_concurrent(cuda):
    """Four short compresses on four streams at once, repeated: byte-identical frames."""
    g = torch.Generator(device=cuda).manual_seed(77)
    xs = [torch.randn(380_000, device=cuda, generator=g) for _ in range(4)]
    refs = [O.compress_frame(_host(x), 50.0, method="threshold") for x in xs]
    streams = [torch.cuda.Stream(device=cuda) for _ in xs]
    prev = _lib.lib().gp_set_cluster_path(2)
    for _ in range(3):
        ps = []
        for x, s in zip(xs, streams):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                ps.append(P.topk_compress(x, 50.0))
        torch.cuda.synchronize()
        assert [p.to_bytes() for p in ps] == refs
    _lib.lib().gp_set_cluster_path(prev)


def test_cluster_default_routing(cuda):
    """Mode 1 (default): vectors up to 98,304 elements take the cluster kernel,
    longer ones the cooperative grid; both bit-exact at the boundary."""
    L = _lib.lib()
    assert L.gp_set_cluster_path(1) in (0, 1, 2)
    g = torch.Generator(device=cuda).manual_seed(9)
    for d in (98_303, 98_304, 98_305):
        x = torch.randn(d, device=cuda, generator=g)
        assert _frame(x, 20.0) == O.compress_frame(_host(x), 20.0, method="threshold"), d
