"""Compressed stage-boundary send/recv: the reference executor's message path on GPUs.

The reference delivers every cross-device OpData through an in-process dict
inbox, compressing on the way (pkg/src/geopipe/executor.py:207-220 and
:248-297):

    payload, shape = _maybe_compress(value, (src, dst), plan)   # :258 / :281
    dest.inbox[key] = _maybe_decompress(payload, shape)          # :270-271 / :293

Here the sender GPU compresses straight into the reference wire frame
(`{d,k} + k*i64 + k*f32`, compressor.py:39-44) with the sm_100a kernel, NCCL
moves the frame over NVLink (torch.distributed P2P, one process per GPU), and
the receiver GPU decompresses the frame in place into its activation buffer.
Both ends size the frame from (d, ratio) alone — k = select_k(d, ratio) is a
pure function — so no size handshake precedes the payload.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist

from . import _lib
from .compressor import CompressionPlan, SparsePayload, _DTYPE_CODE, _Workspace, _stream_handle, select_k, \
    topk_compress, topk_decompress
from .errors import IndexOutOfRange, raise_for_status


def maybe_compress(payload: torch.Tensor, link, plan: Optional[CompressionPlan]):
    """executor.py:207-214 — pass-through without a plan or at ratio <= 1."""
    if plan is None:
        return payload, None
    ratio = plan.ratio_for(*link)
    if ratio <= 1.0:
        return payload, None
    return topk_compress(payload.reshape(-1), ratio), tuple(payload.shape)


def maybe_decompress(payload, shape):
    """executor.py:217-220."""
    if shape is None:
        return payload
    return topk_decompress(payload).reshape(shape)


def frame_bytes(d: int, ratio: float) -> int:
    return 16 + 12 * select_k(d, ratio)


# ---------------------------------------------------------------------------
# OpData envelope (opdag.py:67-86): the reference routes every cross-device
# payload in an OpData carrying the producer, consumers, iteration,
# micro-batch and compress_cfg {algo, shape} (executor.py:259-268, :283-292).
# Here a 128-byte envelope of 16 int64 travels ahead of each stage-boundary
# message in the same buffer, written and checked on the device.

ENVELOPE_BYTES = _lib.ENVELOPE_BYTES
ENVELOPE_MAGIC = 0x41504F4441544131  # "1ATADOPA": an OpData envelope, layout version 1
KIND_ACTIVATION, KIND_GRADIENT = 0, 1
ENVELOPE_ALL = (1 << _lib.ENVELOPE_WORDS) - 1


def envelope_fields(step: int, micro_batch: int, src: int, dst: int, kind: int, compressed: bool,
                    payload_bytes: int, shape) -> list:
    """[magic, iteration (local_iter), micro_batch, src stage, dst stage, kind (0 activation, 1
    gradient), compressed (compress_cfg algo 'topk'), payload bytes, ndim, shape[4], 0, 0, 0]."""
    shape = [int(v) for v in shape]
    if len(shape) > 4:
        shape = shape[:3] + [int(math.prod(shape[3:]))]
    return ([ENVELOPE_MAGIC, int(step), int(micro_batch), int(src), int(dst), int(kind), int(bool(compressed)),
             int(payload_bytes), len(shape)] + shape + [0] * (4 - len(shape)) + [0, 0, 0])


def write_envelope(buf: torch.Tensor, fields: list) -> None:
    """Write the envelope into the first 128 bytes of a uint8 message buffer (stream-ordered on a GPU)."""
    if buf.is_cuda:
        with torch.cuda.device(buf.device):
            st = _lib.lib().gp_envelope_write(buf.data_ptr(), (ctypes.c_int64 * _lib.ENVELOPE_WORDS)(*fields),
                                              _stream_handle(buf.device))
        raise_for_status(st, "gp_envelope_write")
    else:
        buf[:ENVELOPE_BYTES].view(torch.int64).copy_(torch.tensor(fields, dtype=torch.int64))


def check_envelope(buf: torch.Tensor, expected: list, err: Optional[torch.Tensor] = None,
                   mask: int = ENVELOPE_ALL) -> None:
    """Compare a received envelope with the receiver's expectation: on a GPU a
    stream-ordered check raising GP_FLAG_ENVELOPE in `err` (read at the step's
    flag check); on CPU ranks at once (ValueError)."""
    if buf.is_cuda:
        with torch.cuda.device(buf.device):
            st = _lib.lib().gp_envelope_check(buf.data_ptr(), (ctypes.c_int64 * _lib.ENVELOPE_WORDS)(*expected),
                                              mask, err.data_ptr(), _stream_handle(buf.device))
        raise_for_status(st, "gp_envelope_check")
        return
    got = buf[:ENVELOPE_BYTES].view(torch.int64).tolist()
    bad = [i for i in range(_lib.ENVELOPE_WORDS) if (mask >> i) & 1 and got[i] != expected[i]]
    if bad:
        raise ValueError(f"message envelope fields {bad} are {[got[i] for i in bad]}, expected "
                         f"{[expected[i] for i in bad]}")


@dataclass
class FrameCodec:
    """Device-side compress-to-frame / decompress-from-frame with reusable buffers.

    The hot path of a pipeline stage boundary: no host synchronisation.  Every
    decompress checks the received frame on the device (index range, strict
    order, and its {d, k} header against the receiver's own (d, k)); failures
    accumulate in a device flag that `check()` reads once per step.
    """

    device: torch.device

    def __post_init__(self):
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)

    def compress(self, x: torch.Tensor, ratio: float, frame: Optional[torch.Tensor] = None) -> torch.Tensor:
        with torch.cuda.device(self.device):
            return self._compress(x, ratio, frame)

    def _compress(self, x: torch.Tensor, ratio: float, frame: Optional[torch.Tensor]) -> torch.Tensor:
        flat = x.reshape(-1)
        if not flat.is_contiguous():
            flat = flat.contiguous()
        d = flat.numel()
        k = select_k(d, ratio)
        if frame is None:
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=self.device)
        code = _DTYPE_CODE[flat.dtype]
        sp = _stream_handle(self.device)
        ws, wsb = _Workspace.get(self.device, sp, d, code)
        st = _lib.lib().gp_topk_compress_frame(flat.data_ptr(), code, d, k, frame.data_ptr(), ws, wsb, sp)
        raise_for_status(st, "gp_topk_compress_frame", ratio)
        return frame

    def decompress(self, frame: torch.Tensor, out: torch.Tensor, ratio: float, accumulate: bool = False):
        with torch.cuda.device(self.device):
            return self._decompress(frame, out, ratio, accumulate)

    def _decompress(self, frame: torch.Tensor, out: torch.Tensor, ratio: float, accumulate: bool):
        d = out.numel()
        k = select_k(d, ratio)
        st = _lib.lib().gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), _DTYPE_CODE[out.dtype],
                                                 1 if accumulate else 0, self.err.data_ptr(),
                                                 _stream_handle(self.device))
        raise_for_status(st, "gp_topk_decompress_frame")
        return out

    # ---- device-resident k (north_star item 4): k comes from device memory
    # (e.g. the on-device Eq. 6 plan), frames are sized for a host-known
    # capacity k_cap, and the receiver reads k from the frame header.

    def compress_dk(self, x: torch.Tensor, k_dev: torch.Tensor, k_cap: int,
                    frame: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Compress with k = k_dev[0] (int64 CUDA scalar) into a 16 + 12*k_cap byte frame."""
        with torch.cuda.device(self.device):
            flat = x.reshape(-1)
            if not flat.is_contiguous():
                flat = flat.contiguous()
            d = flat.numel()
            if frame is None:
                frame = torch.empty(16 + 12 * k_cap, dtype=torch.uint8, device=self.device)
            code = _DTYPE_CODE[flat.dtype]
            sp = _stream_handle(self.device)
            ws, wsb = _Workspace.get(self.device, sp, d, code)
            st = _lib.lib().gp_topk_compress_frame_dk(flat.data_ptr(), code, d, k_dev.data_ptr(), k_cap,
                                                      frame.data_ptr(), self.err.data_ptr(), ws, wsb, sp, 0)
            raise_for_status(st, "gp_topk_compress_frame_dk")
            return frame

    def decompress_dk(self, frame: torch.Tensor, out: torch.Tensor, k_cap: int, accumulate: bool = False):
        """Decompress a frame whose k is read from its own header (1 <= k <= k_cap)."""
        with torch.cuda.device(self.device):
            st = _lib.lib().gp_topk_decompress_frame_dk(frame.data_ptr(), out.numel(), k_cap, out.data_ptr(),
                                                        _DTYPE_CODE[out.dtype], 1 if accumulate else 0,
                                                        self.err.data_ptr(), _stream_handle(self.device))
            raise_for_status(st, "gp_topk_decompress_frame_dk")
            return out

    def check(self):
        """Read the accumulated device flag (one host sync) and raise on any failure."""
        flag = int(self.err.item())
        if flag:
            self.err.zero_()
        if flag & _lib.FLAG_OUT_OF_RANGE:
            raise IndexOutOfRange("received frame holds an index outside [0, d)")
        if flag & _lib.FLAG_UNSORTED:
            raise ValueError("received frame indices are not strictly increasing")
        if flag & _lib.FLAG_HEADER:
            raise ValueError("received frame header {d, k} disagrees with the receiver's (d, k)")
        if flag & _lib.FLAG_BAD_K:
            raise ValueError("device-resident k outside [1, min(k_cap, d)]")
        if flag & _lib.FLAG_ENVELOPE:
            raise ValueError("a received message's OpData envelope differs from the receiver's expectation")


class StageLink:
    """Compressed channels between pipeline ranks (one process per GPU).

    `exchange` compresses every outgoing tensor into a reference wire frame on
    the sender's current stream, posts all sends and receives as one NCCL
    group (`batch_isend_irecv`, so neighbouring stages cannot deadlock),
    waits, and decompresses every received frame into its destination buffer.
    The codec is pluggable (default: the sm_100a `FrameCodec`); frame sizes are
    derived from (d, ratio) on both ends, and each received frame's header is
    checked against them on the device.  With `check=True` (default) the
    codec's flag is read once at the end of the exchange (one host sync per
    exchange, not per frame) and a corrupt or mismatched frame raises.
    """

    def __init__(self, device: torch.device, group=None, codec=None):
        self.device = device
        self.group = group
        self.codec = codec if codec is not None else FrameCodec(device)

    def exchange(self, sends, recvs, check: bool = True):
        """sends: [(tensor, ratio, dst)]; recvs: [(out_tensor, ratio, src)] -> decompressed outs."""
        ops, frames_in = [], []
        for x, ratio, dst in sends:
            if ratio <= 1.0:
                ops.append(dist.P2POp(dist.isend, x.contiguous(), dst, group=self.group))
            else:
                ops.append(dist.P2POp(dist.isend, self.codec.compress(x, ratio), dst, group=self.group))
        for out, ratio, src in recvs:
            if ratio <= 1.0:
                buf = out
            else:
                buf = torch.empty(frame_bytes(out.numel(), ratio), dtype=torch.uint8, device=out.device)
            frames_in.append(buf)
            ops.append(dist.P2POp(dist.irecv, buf, src, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        outs = []
        for (out, ratio, _src), buf in zip(recvs, frames_in):
            if ratio > 1.0:
                self.codec.decompress(buf, out, ratio)
            outs.append(out)
        if check and hasattr(self.codec, "check"):
            self.codec.check()
        return outs


def payload_from_frame(frame: torch.Tensor, values_dtype=torch.float32) -> SparsePayload:
    """View a device frame as a SparsePayload (float32 values, like the wire)."""
    d, k = (int(v) for v in frame[:16].view(torch.int64).tolist())
    idx = frame[16:16 + 8 * k].view(torch.int64)
    vals = frame[16 + 8 * k:16 + 12 * k].view(torch.float32)
    if values_dtype != torch.float32:
        vals = vals.to(values_dtype)
    return SparsePayload(values=vals, indices=idx, original_len=d, frame=frame)


__all__ = ["maybe_compress", "maybe_decompress", "frame_bytes", "FrameCodec", "StageLink", "payload_from_frame",
           "ENVELOPE_BYTES", "envelope_fields", "write_envelope", "check_envelope", "KIND_ACTIVATION", "KIND_GRADIENT"]
