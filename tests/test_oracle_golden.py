"""Pin the CPU oracle to the reference's own outputs (CPU only, no GPU).

Every golden frame in tests/golden/golden.npz was produced by
geopipe.compressor itself (tests/golden/make_golden.py).  The oracle must
reproduce each one byte-for-byte, with both of its selection restatements.
"""
import numpy as np
import pytest

from golden_cases import cases, plans
from oracle import compressor_oracle as O


@pytest.mark.parametrize("prefix", ["f32", "f64"])
def test_oracle_argsort_matches_reference_frames(prefix):
    n = 0
    for name, x, ratio, frame in cases(prefix):
        assert O.compress_frame(x, ratio, "argsort") == frame, name
        n += 1
    assert n > 10


@pytest.mark.parametrize("prefix", ["f32", "f64"])
def test_oracle_threshold_matches_reference_frames(prefix):
    for name, x, ratio, frame in cases(prefix):
        assert O.compress_frame(x, ratio, "threshold") == frame, name


def test_oracle_bf16_is_reference_on_upcast():
    for name, bits, ratio, frame in cases("bf16"):
        up = O.bf16_bits_to_f32(bits)
        assert O.compress_frame(up, ratio, "threshold") == frame, name


def test_oracle_round_trip_and_decompress():
    for name, x, ratio, frame in list(cases("f32"))[:300]:
        vals, idx, d = O.from_bytes(frame)
        dense = O.topk_decompress(vals, idx, d)
        assert dense.dtype == np.float64 and dense.size == d
        # the golden frame decodes to the oracle's own decompress of a fresh
        # compress, bit for bit (values widened to float64 as from_bytes does)
        v2, i2, _ = O.topk_compress(x, ratio)
        ref = O.topk_decompress(v2, i2, d).astype(np.float64)
        assert np.array_equal(dense.view(np.uint64), ref.view(np.uint64)), name
        np.testing.assert_array_equal(dense[idx], x[idx].astype(np.float64))


def test_oracle_plans_match_reference():
    for R, r, expected in plans():
        got = O.adatopk_ratios({i: v for i, v in enumerate(R)}, r)
        assert [got[i] for i in range(len(R))] == expected


def test_oracle_errors():
    with pytest.raises(O.EmptyVector):
        O.topk_compress([], 2)
    with pytest.raises(O.InvalidRatio):
        O.select_k(10, 0.5)
    with pytest.raises(O.IndexOutOfRange):
        O.topk_decompress(np.ones(1), np.array([5]), 3)
    with pytest.raises(O.NoCommunication):
        O.adatopk_ratios({"a": 0.0}, 10)


def test_rank_key_order_matches_numpy_sort():
    """The integer key realises numpy's -|x| stable order, NaN last."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(5000).astype(np.float32)
    x[rng.choice(5000, 300, replace=False)] = rng.choice(
        np.array([np.nan, np.inf, -np.inf, 0.0, -0.0, 1e-45, -1e-45], dtype=np.float32), 300)
    order_ref = np.argsort(-np.abs(x), kind="stable")
    keys = O.rank_keys(x)
    order_key = np.lexsort((np.arange(x.size), -keys.astype(np.int64)))
    np.testing.assert_array_equal(order_ref, order_key)
