"""B200 drop-in for `geopipe.compressor` (reference: pkg/src/geopipe/compressor.py).

Same module-level names, argument meaning and exceptions as the reference:

    VALUE_BYTES, INDEX_BYTES, SPARSE_EXPANSION         (compressor.py:14-17)
    SparsePayload(values, indices, original_len)       (:20-53)
    CompressionPlan(base_ratio, per_link, R_estimates) (:56-70)
    select_k, topk_compress, topk_decompress, wire_bytes,
    adatopk_plan, uniform_plan, per_device_ratios      (:73-150)

What changes is where the work happens: `topk_compress` / `topk_decompress`
run the sm_100a kernels of libadatopk.so on the current CUDA device and
stream (tensors stay in HBM; host inputs are copied in first).  Payload
tensors are CUDA tensors; `SparsePayload.to_bytes()` is byte-identical to the
reference frame.  There is no CPU fallback: without a CUDA device the compute
entry points raise.
"""
from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import EmptyVector, IndexOutOfRange, InvalidRatio, NoCommunication, raise_for_status

VALUE_BYTES = 4   # float32 values on the wire
INDEX_BYTES = 8   # int64 indices on the wire
SPARSE_EXPANSION = (VALUE_BYTES + INDEX_BYTES) / VALUE_BYTES

_DTYPE_CODE = {torch.float32: _lib.DTYPE_F32, torch.bfloat16: _lib.DTYPE_BF16, torch.float64: _lib.DTYPE_F64}


# ---------------------------------------------------------------------------
# payload


@dataclass
class SparsePayload:
    """Kept entries of one compressed vector (mirror of compressor.py:20-53).

    `values` (input dtype) and `indices` (int64, strictly increasing) are CUDA
    tensors.  `frame`, when present, is the device copy of the reference wire
    frame `{d:u64,k:u64} + k*i64 + k*f32`; for float32 inputs `indices` and
    `values` are views into it.
    """

    values: torch.Tensor
    indices: torch.Tensor
    original_len: int
    frame: Optional[torch.Tensor] = field(default=None, repr=False, compare=False)
    # set when the frame was written together with these fields (by the
    # compress kernel or by from_bytes): (indices, its _version, values, its
    # _version, original_len).  While all of these still hold, the payload is
    # unmodified: to_bytes() may return the cached frame, and for kernel-made
    # payloads topk_decompress need not read its validation flag back (the
    # indices are strictly increasing and in range by construction).  Any
    # replaced field (dataclasses.replace included), in-place write (views
    # share the version counter) or new original_len invalidates it.
    _produced: Optional[tuple] = field(default=None, repr=False, compare=False)
    _kernel_made: bool = field(default=False, repr=False, compare=False)

    @property
    def k(self) -> int:
        return int(self.values.numel())

    @property
    def ratio_used(self) -> float:
        return self.original_len / self.k

    @property
    def payload_nbytes(self) -> int:
        """Wire accounting for the values+indices body (excludes the 16B header)."""
        return self.k * (VALUE_BYTES + INDEX_BYTES)

    def _unmodified(self) -> bool:
        p = self._produced
        return (p is not None and self.indices is p[0] and self.indices._version == p[1] and self.values is p[2]
                and self.values._version == p[3] and int(self.original_len) == p[4])

    def to_bytes(self) -> bytes:
        """Little-endian frame: {d: u64, k: u64}, k x i64 indices, k x f32 values.

        Always the current fields: the cached device frame when the payload is
        unmodified, else a frame packed on the device (gp_pack_frame) from the
        fields as they are now."""
        if self.frame is not None and self._unmodified():
            return self.frame.cpu().numpy().tobytes()
        values, indices = self.values, self.indices
        if not (isinstance(values, torch.Tensor) and values.is_cuda):
            raise TypeError("SparsePayload.values must be a CUDA tensor")
        device = values.device
        vals = values.reshape(-1).contiguous()
        idx = torch.as_tensor(indices, device=device).reshape(-1).contiguous()
        k = int(vals.numel())
        if idx.numel() != k:
            raise ValueError(f"payload has {k} values but {idx.numel()} indices")
        if idx.dtype not in (torch.int64, torch.int32):
            idx = idx.to(torch.int64)
        code = _DTYPE_CODE.get(vals.dtype)
        if code is None:
            vals, code = vals.to(torch.float64), _lib.DTYPE_F64  # exact widening of other float/int dtypes
        frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=device)
        with torch.cuda.device(device):
            st = _lib.lib().gp_pack_frame(idx.data_ptr(), idx.element_size(), vals.data_ptr(), code, k,
                                          int(self.original_len), frame.data_ptr(), _stream_handle(device))
        raise_for_status(st, "gp_pack_frame")
        return frame.cpu().numpy().tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes, device=None) -> "SparsePayload":
        """Parse a frame; like the reference (compressor.py:46-53) values come back as float64.

        The frame is uploaded once and unpacked on the device (gp_unpack_frame);
        a buffer shorter than its header's k says raises ValueError, as numpy's
        `frombuffer(count=k)` does in the reference."""
        if len(raw) < 16:
            raise ValueError(f"frame of {len(raw)} bytes has no 16-byte header")
        d, k = struct.unpack_from("<QQ", raw, 0)
        if len(raw) < 16 + 12 * k:
            raise ValueError(f"frame of {len(raw)} bytes is shorter than its header's k = {k} entries need")
        dev = _device(device)
        frame = torch.frombuffer(bytearray(raw[: 16 + 12 * k]), dtype=torch.uint8).to(dev)
        indices = torch.empty(k, dtype=torch.int64, device=dev)
        values = torch.empty(k, dtype=torch.float64, device=dev)
        err = _Flags.get(dev, _stream_handle(dev))
        with torch.cuda.device(dev):
            st = _lib.lib().gp_unpack_frame(frame.data_ptr(), k, d, indices.data_ptr(), values.data_ptr(),
                                            _lib.DTYPE_F64, None, err.data_ptr(), _stream_handle(dev))
        raise_for_status(st, "gp_unpack_frame")
        p = cls(values=values, indices=indices, original_len=int(d), frame=frame)
        p._produced = (indices, indices._version, values, values._version, int(d))
        return p


@dataclass
class CompressionPlan:
    """Per-link ratios (mirror of compressor.py:56-70)."""

    base_ratio: float
    per_link: dict                      # (src, dst) -> ratio >= 1
    R_estimates: dict = field(default_factory=dict)

    def ratio_for(self, src, dst) -> float:
        return self.per_link.get((src, dst), 1.0)

    def to_dict(self) -> dict:
        # The reference sorts R_estimates' mixed tuple/str keys and raises
        # TypeError for adaptive plans (SURVEY.md §7 hard part 11); sort by the
        # string form instead so the dict is always produced.
        return {
            "base_ratio": self.base_ratio,
            "per_link": {f"{s}->{d}": r for (s, d), r in sorted(self.per_link.items(), key=lambda kv: str(kv[0]))},
            "R_estimates": {str(k): v for k, v in sorted(self.R_estimates.items(), key=lambda kv: str(kv[0]))},
        }


# ---------------------------------------------------------------------------
# k and wire size (pure host arithmetic, identical to the reference)


def select_k(d: int, ratio: float) -> int:
    """k = max(1, floor(d / ratio)); compressor.py:73-76."""
    if ratio < 1:
        raise InvalidRatio(ratio)
    return max(1, math.floor(d / ratio))


def wire_bytes(d: int, ratio: float) -> int:
    """12 bytes per kept entry; compressor.py:106-108."""
    return select_k(d, ratio) * (VALUE_BYTES + INDEX_BYTES)


# ---------------------------------------------------------------------------
# device plumbing


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the AdaTopK compressor runs on a CUDA device (sm_100a); no CPU fallback exists")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise RuntimeError(f"AdaTopK tensors must live on a CUDA device, got {device}")
    return device if device.index is not None else torch.device("cuda", torch.cuda.current_device())


def _stream_handle(device: torch.device, stream=None) -> int:
    """The raw cudaStream_t of `stream` (None: the current stream of `device`)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


class _Workspace:
    """Per (device, stream) scratch for gp_topk_compress, zeroed once, grown on demand.

    The state region's extent depends only on the buffer size
    (include/adatopk.h), so one buffer serves every vector that fits it."""

    _cache: dict = {}

    @classmethod
    def get(cls, device: torch.device, stream_ptr: int, d: int, dtype_code: int) -> tuple[int, int]:
        need = int(_lib.lib().gp_topk_workspace_bytes(d, dtype_code))
        key = (device.index, stream_ptr)
        buf = cls._cache.get(key)
        if buf is None or buf.numel() < need:
            buf = torch.empty(need, dtype=torch.uint8, device=device)
            raise_for_status(_lib.lib().gp_workspace_init(buf.data_ptr(), need, stream_ptr), "gp_workspace_init")
            cls._cache[key] = buf
        return buf.data_ptr(), int(buf.numel())

    @classmethod
    def clear(cls) -> None:
        cls._cache.clear()


class _Flags:
    """Per (device, stream) asynchronous validation flag (one int32), zeroed at
    creation and re-zeroed only after it was read non-zero: no per-call fill."""

    _cache: dict = {}

    @classmethod
    def get(cls, device: torch.device, stream_ptr: int) -> torch.Tensor:
        key = (device.index, stream_ptr)
        f = cls._cache.get(key)
        if f is None:
            f = torch.zeros(1, dtype=torch.int32, device=device)
            cls._cache[key] = f
        return f

    @staticmethod
    def read(flag: torch.Tensor) -> int:
        v = int(flag.item())
        if v:
            flag.zero_()
        return v


def _compute_dtype(dtype: torch.dtype) -> torch.dtype:
    """The kernel dtype an input dtype is ranked in: f32/bf16/f64 as they are,
    float16 as float32 and integers/bool as float64 (exact widenings that keep
    the magnitude order; integers exactly below 2^53)."""
    if dtype in _DTYPE_CODE:
        return dtype
    if dtype.is_floating_point:
        return torch.float32 if torch.finfo(dtype).bits <= 16 else torch.float64
    if dtype.is_complex:
        raise TypeError(f"unsupported dtype {dtype}")
    return torch.float64


def _as_device_flat(vector, device: torch.device):
    """Flatten like `np.asarray(vector).reshape(-1)` (compressor.py:85-87), on
    the device; returns (flat tensor in its kernel dtype, the input's dtype)."""
    if isinstance(vector, torch.Tensor):
        t = vector
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(vector)))
    orig = t.dtype
    if t.device != device:
        t = t.to(device, non_blocking=t.is_pinned())
    t = t.reshape(-1)
    cd = _compute_dtype(orig)
    if cd != orig:
        t = t.to(cd)
    return t.contiguous(), orig


# ---------------------------------------------------------------------------
# compress / decompress


def _on_stream(stream):
    """Run the body on `stream` (None: the current stream): staging copies,
    outputs, the kernels and any flag read are then ordered on that one stream,
    and the caching allocator records their use there."""
    return torch.cuda.stream(stream) if stream is not None else _NullCtx()


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def topk_compress(vector, ratio: float, *, stream=None) -> SparsePayload:
    """Keep the k = max(1, floor(d/ratio)) largest-magnitude entries (compressor.py:79-94).

    Magnitude ties keep the lower index; NaN ranks below every number.  Values
    are stored in index order with their original dtype; the device frame holds
    the f32 wire values.  Runs the cooperative sm_100a select+compact kernel.
    """
    device = _device(vector.device if isinstance(vector, torch.Tensor) and vector.is_cuda else None)
    with torch.cuda.device(device), _on_stream(stream):  # launches go to the tensor's GPU whatever the current device
        return _topk_compress_on(vector, ratio, device)


def _topk_compress_on(vector, ratio: float, device: torch.device) -> SparsePayload:
    flat, orig_dtype = _as_device_flat(vector, device)
    d = flat.numel()
    if d == 0:
        raise EmptyVector("cannot compress a zero-length vector")
    k = select_k(d, ratio)
    code = _DTYPE_CODE.get(flat.dtype)
    if code is None:
        raise TypeError(f"unsupported dtype {flat.dtype}; expected float32, bfloat16 or float64")
    sp = _stream_handle(device)
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=device)
    idx = frame[16:16 + 8 * k].view(torch.int64)
    fvals = frame[16 + 8 * k:].view(torch.float32)
    values = fvals if code == _lib.DTYPE_F32 else torch.empty(k, dtype=flat.dtype, device=device)
    ws_ptr, ws_bytes = _Workspace.get(device, sp, d, code)
    st = _lib.lib().gp_topk_compress(
        flat.data_ptr(), code, d, k, idx.data_ptr(), 8, fvals.data_ptr(), _lib.DTYPE_F32,
        None if code == _lib.DTYPE_F32 else values.data_ptr(), frame.data_ptr(), ws_ptr, ws_bytes, sp)
    raise_for_status(st, "gp_topk_compress", ratio)
    if orig_dtype != values.dtype:  # the reference keeps the input dtype (values = flat[kept].copy())
        values = values.to(orig_dtype)  # exact: every value came from an input of that dtype
    p = SparsePayload(values=values, indices=idx, original_len=d, frame=frame)
    p._produced = (idx, idx._version, values, values._version, d)
    p._kernel_made = True
    return p


def topk_decompress(payload: SparsePayload, *, out: Optional[torch.Tensor] = None, accumulate: bool = False,
                    check: bool = True, stream=None) -> torch.Tensor:
    """Dense length-d vector: kept values at their indices, zero elsewhere (compressor.py:97-103).

    `accumulate=True` adds into `out` instead (residual mode; not in the
    reference; its indices must be strictly increasing, else ValueError).
    With `check=True` (default, reference behaviour) the device validation
    flag is read back and IndexOutOfRange is raised synchronously; unsorted or
    repeated indices are re-run through the general scatter with numpy's
    last-write-wins semantics.  A payload made by topk_compress and not
    modified since is valid by construction, so its flag is not read back (no
    host sync); any other payload is checked.
    """
    values = payload.values
    device = _device(values.device if isinstance(values, torch.Tensor) and values.is_cuda else None)
    with torch.cuda.device(device), _on_stream(stream):  # launches go to the payload's GPU whatever the current device
        return _topk_decompress_on(payload, device, out, accumulate, check)


def _topk_decompress_on(payload, device: torch.device, out, accumulate: bool, check: bool) -> torch.Tensor:
    values, indices = payload.values, payload.indices
    if not isinstance(values, torch.Tensor) or not values.is_cuda:
        values = torch.as_tensor(np.asarray(values)).to(device)
    if not isinstance(indices, torch.Tensor) or not indices.is_cuda:
        indices = torch.as_tensor(np.asarray(indices, dtype=np.int64)).to(device)
    values = values.reshape(-1).contiguous()
    indices = indices.reshape(-1).contiguous()
    if indices.dtype not in (torch.int64, torch.int32):
        indices = indices.to(torch.int64)
    d, k = int(payload.original_len), int(values.numel())
    if indices.numel() != k:  # numpy raises on the shape mismatch in the reference (compressor.py:101-102)
        raise ValueError(f"payload has {k} values but {indices.numel()} indices")
    # the output has the values' dtype (np.zeros(d, values.dtype)); dtypes the
    # kernels do not take (integers, bool, float16) run widened and are cast back
    # exactly at the end
    user_out = out
    if out is not None and (out.numel() != d or not out.is_contiguous()):
        raise ValueError("out must be a contiguous tensor of original_len elements")
    res_dtype = values.dtype if out is None else out.dtype
    if values.dtype not in _DTYPE_CODE:
        values = values.to(_compute_dtype(values.dtype))
    code = _DTYPE_CODE[values.dtype]
    if out is None or out.dtype not in _DTYPE_CODE:
        wd = values.dtype if out is None else _compute_dtype(out.dtype)
        if accumulate:
            out = torch.zeros(d, dtype=wd, device=device) if user_out is None else user_out.to(wd)
        else:
            out = torch.empty(d, dtype=wd, device=device)
    out_code = _DTYPE_CODE[out.dtype]
    if d == 0 and k > 0:
        raise IndexOutOfRange(indices)
    sp = _stream_handle(device)
    err = _Flags.get(device, sp)
    L = _lib.lib()
    ib = indices.element_size()
    # a kernel-made, unmodified payload is valid by construction: no sortedness
    # scan on the device (GP_DECOMPRESS_TRUSTED) and no flag read on the host
    trusted = getattr(payload, "_kernel_made", False) and payload._unmodified()
    st = L.gp_topk_decompress(indices.data_ptr(), ib, values.data_ptr(), code, k, d, out.data_ptr(), out_code,
                              (1 if accumulate else 0) | (2 if trusted else 0), err.data_ptr(), sp)
    raise_for_status(st, "gp_topk_decompress", indices)
    if trusted:
        check = False
    if check:
        flag = _Flags.read(err)
        if flag & _lib.FLAG_UNSORTED:
            if accumulate:
                raise ValueError("residual-mode decompress needs strictly increasing indices")
            scratch = torch.empty(max(d, 1), dtype=torch.int32, device=device)
            st = L.gp_topk_decompress_unsorted(indices.data_ptr(), ib, values.data_ptr(), code, k, d, out.data_ptr(),
                                               out_code, scratch.data_ptr(), err.data_ptr(), sp)
            raise_for_status(st, "gp_topk_decompress_unsorted", indices)
            flag = _Flags.read(err)
        if flag & _lib.FLAG_OUT_OF_RANGE:
            raise IndexOutOfRange(indices)
    if out.dtype != res_dtype:  # widened run: back to the values' (or the caller's out) dtype
        if user_out is not None:
            user_out.copy_(out)
            return user_out
        return out.to(res_dtype)
    return out


# ---------------------------------------------------------------------------
# AdaTopK plans (Eq. 6)


def _plan_arrays(R: list, base_ratio: float, d_per_link=None):
    n = len(R)
    Ra = (ctypes.c_double * max(n, 1))(*R)
    ra = (ctypes.c_double * max(n, 1))()
    if d_per_link is None:
        return Ra, ra, None, None
    da = (ctypes.c_int64 * max(n, 1))(*d_per_link)
    ka = (ctypes.c_int64 * max(n, 1))()
    return Ra, ra, da, ka


def adatopk_plan(stage_costs, cross_link_R: dict, base_ratio: float) -> CompressionPlan:
    """Per-link ratios r_i = max(1, 3r * R_i / max R) (compressor.py:111-129).

    The arithmetic runs in the library's host twin of the device kernel
    (gp_adatopk_plan_host), so host plans and on-device plans are the same
    IEEE-double computation.
    """
    if base_ratio < 1:
        raise InvalidRatio(base_ratio)
    links = list(cross_link_R.keys())
    R = [float(cross_link_R[l]) for l in links]
    Ra, ra, _, _ = _plan_arrays(R, base_ratio)
    st = _lib.lib().gp_adatopk_plan_host(Ra, len(R), float(base_ratio), None, ra, None)
    raise_for_status(st, "adatopk_plan", base_ratio)
    per_link = {l: float(ra[i]) for i, l in enumerate(links)}
    estimates = dict(cross_link_R)
    if stage_costs is not None:
        estimates.update({d: stage_costs.receive[d] for d in stage_costs.devices})
    return CompressionPlan(base_ratio=base_ratio, per_link=per_link, R_estimates=estimates)


def adatopk_plan_device(R: torch.Tensor, base_ratio: float, d_per_link: torch.Tensor, *, stream=None):
    """On-device Eq. 6 + select_k: returns (r, k, status) CUDA tensors without a host sync.

    `R` (float64) can be produced on the device, e.g. measured link times, so
    both ends of a link can agree on k without a host round trip.
    """
    device = _device(R.device)
    R = R.to(device=device, dtype=torch.float64).contiguous()
    d_per_link = d_per_link.to(device=device, dtype=torch.int64).contiguous()
    n = R.numel()
    r = torch.empty(n, dtype=torch.float64, device=device)
    k = torch.empty(n, dtype=torch.int64, device=device)
    status = torch.empty(1, dtype=torch.int32, device=device)
    P = ctypes.POINTER
    st = _lib.lib().gp_adatopk_plan(
        ctypes.cast(R.data_ptr(), P(ctypes.c_double)), n, float(base_ratio),
        ctypes.cast(d_per_link.data_ptr(), P(ctypes.c_int64)), ctypes.cast(r.data_ptr(), P(ctypes.c_double)),
        ctypes.cast(k.data_ptr(), P(ctypes.c_int64)), ctypes.cast(status.data_ptr(), P(ctypes.c_int32)),
        _stream_handle(device, stream))
    raise_for_status(st, "gp_adatopk_plan")
    return r, k, status


def uniform_plan(cross_links, base_ratio: float) -> CompressionPlan:
    """Every cross-device link at the base ratio (compressor.py:132-139)."""
    if base_ratio < 1:
        raise InvalidRatio(base_ratio)
    return CompressionPlan(base_ratio=base_ratio, per_link={link: float(base_ratio) for link in cross_links})


def per_device_ratios(plan: Optional[CompressionPlan], devices) -> dict:
    """Receiver-side collapse, min ratio per destination (compressor.py:142-150)."""
    out = {d: 1.0 for d in devices}
    if plan is None:
        return out
    for (_, dst), r in plan.per_link.items():
        if dst in out:
            out[dst] = r if out[dst] == 1.0 else min(out[dst], r)
    return out


__all__ = [
    "VALUE_BYTES", "INDEX_BYTES", "SPARSE_EXPANSION", "SparsePayload", "CompressionPlan", "select_k",
    "topk_compress", "topk_decompress", "wire_bytes", "adatopk_plan", "adatopk_plan_device", "uniform_plan",
    "per_device_ratios", "InvalidRatio", "EmptyVector", "IndexOutOfRange", "NoCommunication",
]
