"""CPU oracle for the AdaTopK hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` leg may import this module, and only as the checker or the
timed CPU reference — never as part of the product path (the product is the
sm_100a library behind paper_2410_12707_b200.compressor, which has no CPU
fallback).

It restates, in NumPy, the reference compressor
(/root/reference/pkg/src/geopipe/compressor.py) function by function; each
function cites the lines it follows.  Parity status: PINNED — the restatement
is checked byte-for-byte against golden frames produced by the reference
itself (tests/golden/make_golden.py imports geopipe.compressor in the build
container and stores its outputs; tests/test_oracle_golden.py replays them).

Conventions restated here:
  * k = max(1, floor(d / ratio)), ratio < 1 -> InvalidRatio        (:73-76)
  * selection = stable argsort of -|x|, first k, sorted ascending (:91-93);
    NumPy sorts NaN last and keeps ties in index order
  * values keep the input dtype (:94); the wire frame casts them to <f4 (:43)
  * decompress = zeros(d, values.dtype); out[indices] = values     (:97-103)
  * Eq. 6: r_i = max(1.0, 3.0 * r * R_i / max R), left to right    (:111-129)
  * bf16 inputs: the reference applied to the exact float32 upcast
"""
from __future__ import annotations

import math
import struct

import numpy as np


class OracleError(Exception):
    pass


class InvalidRatio(OracleError):
    pass


class EmptyVector(OracleError):
    pass


class IndexOutOfRange(OracleError):
    pass


class NoCommunication(OracleError):
    pass


VALUE_BYTES = 4
INDEX_BYTES = 8


def select_k(d: int, ratio: float) -> int:
    """compressor.py:73-76."""
    if ratio < 1:
        raise InvalidRatio(ratio)
    return max(1, math.floor(d / ratio))


def wire_bytes(d: int, ratio: float) -> int:
    """compressor.py:106-108."""
    return select_k(d, ratio) * (VALUE_BYTES + INDEX_BYTES)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact bf16 -> f32 upcast of raw uint16 bit patterns."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def topk_indices_argsort(flat: np.ndarray, k: int) -> np.ndarray:
    """The reference selection verbatim in spirit: compressor.py:91-93."""
    order = np.argsort(-np.abs(flat), kind="stable")
    return np.sort(order[:k]).astype(np.int64)


def rank_keys(flat: np.ndarray) -> np.ndarray:
    """Integer rank key of the reference total order: NaN -> 0, else |bits| + 1.

    Equivalent to ordering by -|x| with NaN last (SURVEY.md §7 hard part 1).
    """
    if flat.dtype == np.float32:
        a = flat.view(np.uint32) & np.uint32(0x7FFFFFFF)
        return np.where(a > np.uint32(0x7F800000), np.uint32(0), a + np.uint32(1)).astype(np.uint64)
    if flat.dtype == np.float64:
        a = flat.view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
        return np.where(a > np.uint64(0x7FF0000000000000), np.uint64(0), a + np.uint64(1))
    raise TypeError(flat.dtype)


def topk_indices_threshold(flat: np.ndarray, k: int) -> np.ndarray:
    """Same selection, restated as threshold + tie quota (O(d) with np.partition).

    T = k-th largest key; keep every key > T and the first (k - #{key > T})
    keys == T in index order.  Used for large d; cross-checked against
    topk_indices_argsort in tests.
    """
    keys = rank_keys(flat)
    d = keys.size
    T = np.partition(keys, d - k)[d - k]
    gt = keys > T
    need = k - int(gt.sum())
    eq_idx = np.flatnonzero(keys == T)[:need]
    sel = gt
    sel[eq_idx] = True
    return np.flatnonzero(sel).astype(np.int64)


def topk_compress(vector, ratio: float, method: str = "argsort"):
    """compressor.py:79-94 -> (values, indices, d)."""
    flat = np.asarray(vector).reshape(-1)
    d = flat.size
    if d == 0:
        raise EmptyVector("cannot compress a zero-length vector")
    k = select_k(d, ratio)
    kept = topk_indices_argsort(flat, k) if method == "argsort" else topk_indices_threshold(flat, k)
    return flat[kept].copy(), kept, d


def topk_decompress(values: np.ndarray, indices: np.ndarray, d: int) -> np.ndarray:
    """compressor.py:97-103."""
    if len(values) and (indices.min() < 0 or indices.max() >= d):
        raise IndexOutOfRange(indices)
    out = np.zeros(d, dtype=np.asarray(values).dtype)
    out[indices] = values
    return out


def to_bytes(values: np.ndarray, indices: np.ndarray, d: int) -> bytes:
    """SparsePayload.to_bytes, compressor.py:39-44."""
    head = struct.pack("<QQ", d, len(values))
    return (head + np.ascontiguousarray(indices, dtype="<i8").tobytes()
            + np.ascontiguousarray(values, dtype="<f4").tobytes())


def from_bytes(raw: bytes):
    """SparsePayload.from_bytes, compressor.py:46-53 -> (values f64, indices i64, d)."""
    d, k = struct.unpack_from("<QQ", raw, 0)
    idx = np.frombuffer(raw, dtype="<i8", count=k, offset=16).astype(np.int64)
    vals = np.frombuffer(raw, dtype="<f4", count=k, offset=16 + 8 * k).astype(np.float64)
    return vals, idx, d


def compress_frame(vector, ratio: float, method: str = "argsort") -> bytes:
    values, idx, d = topk_compress(vector, ratio, method)
    return to_bytes(values, idx, d)


def adatopk_ratios(cross_link_R: dict, base_ratio: float) -> dict:
    """Eq. 6 per-link ratios, compressor.py:118-125."""
    if base_ratio < 1:
        raise InvalidRatio(base_ratio)
    r_max = max(cross_link_R.values(), default=0.0)
    if r_max <= 0:
        raise NoCommunication("all link communication estimates are zero")
    return {link: max(1.0, 3.0 * base_ratio * r / r_max) for link, r in cross_link_R.items()}
