"""Stage-boundary frames over peer memory (NVLink / NVSwitch), one process per GPU.

The reference delivers every compressed cross-device payload through an
in-process inbox (pkg/src/geopipe/executor.py:248-297).  Here a rank copies its
wire frames straight into its successor's receive buffer with the copy engines
(`cudaMemcpyAsync` to a CUDA-IPC-mapped peer pointer: no SMs are used, so the
transfer of frame i overlaps the compress kernel of frame i+1) and signals an
interprocess event the successor's stream waits on before decompressing.

`PeerRing` is the ring used by the pipeline benchmark (rank r -> r+1):

    ring = PeerRing(recv_bytes, device, cpu_group)
    ring.wait_consumed(stream, parity)   # successor finished with buffer `parity`
    ...copies to ring.peer_recv[parity] + offset (copy stream, stream-ordered)...
    ring.signal_sent(stream)             # after the copies
    cpu_barrier()                        # every rank has recorded its event
    ring.wait_sent(stream)               # predecessor's copies have landed
    ...decompress from ring.recv[parity] + offset...
    ring.signal_consumed(stream)

In pull mode (`PeerRing(..., pull=True)`) nothing is copied: a rank compresses
into its own exported buffer and its successor's decompress kernels read the
frames from it over NVLink; the same events order the two sides.

Handles (buffers and events) are exchanged once over a CPU (gloo) group.  The
receive buffer is double-buffered by step parity: a sender writing buffer p at
step s waits for the consumer's record of step s-2 or later, which every rank
has made before the CPU barrier of step s-1.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .errors import raise_for_status


def _handle(raw: bytes):
    buf = (ctypes.c_char * _lib.IPC_HANDLE_BYTES).from_buffer_copy(raw)
    return buf


class PeerRing:
    """`pull=False` (push): each rank maps its successor's buffer and writes
    frames there (`peer_recv`); it decompresses from its own (`recv`).
    `pull=True`: each rank compresses into its own buffer (`recv` = the local
    frames) and maps its predecessor's (`peer_recv`), which its decompress
    kernels read directly over NVLink: no copy at all.  The events and their
    meaning are the same in both directions."""

    def __init__(self, recv_bytes: int, device: torch.device, cpu_group=None, pull: bool = False):
        L = _lib.lib()
        self.L = L
        self.device = device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if self.world < 2:
            raise ValueError("PeerRing needs at least two ranks")
        self.recv_bytes = (int(recv_bytes) + 255) // 256 * 256
        with torch.cuda.device(device):
            self.recv_base = ctypes.c_void_p()
            raise_for_status(L.gp_peer_alloc(2 * self.recv_bytes, ctypes.byref(self.recv_base)), "gp_peer_alloc")
            mh = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
            raise_for_status(L.gp_ipc_mem_handle(self.recv_base, mh), "gp_ipc_mem_handle")
            self.sent, self.consumed = ctypes.c_void_p(), ctypes.c_void_p()
            sh = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
            ch = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
            raise_for_status(L.gp_ipc_event_create(ctypes.byref(self.sent), sh), "gp_ipc_event_create")
            raise_for_status(L.gp_ipc_event_create(ctypes.byref(self.consumed), ch), "gp_ipc_event_create")
            objs = [None] * self.world
            dist.all_gather_object(objs, (bytes(mh), bytes(sh), bytes(ch)), group=cpu_group)
            nxt, prv = (self.rank + 1) % self.world, (self.rank - 1) % self.world
            self.pull = bool(pull)
            self.peer_base = ctypes.c_void_p()
            raise_for_status(L.gp_ipc_open_mem(_handle(objs[prv if self.pull else nxt][0]),
                                               ctypes.byref(self.peer_base)), "gp_ipc_open_mem")
            self.prev_sent, self.next_consumed = ctypes.c_void_p(), ctypes.c_void_p()
            raise_for_status(L.gp_ipc_open_event(_handle(objs[prv][1]), ctypes.byref(self.prev_sent)),
                             "gp_ipc_open_event")
            raise_for_status(L.gp_ipc_open_event(_handle(objs[nxt][2]), ctypes.byref(self.next_consumed)),
                             "gp_ipc_open_event")

    # device pointers of buffer `parity`: the local one / the mapped peer's
    # (push: the successor's receive buffer; pull: the predecessor's frames)
    def recv(self, parity: int) -> int:
        return self.recv_base.value + (parity & 1) * self.recv_bytes

    def peer_recv(self, parity: int) -> int:
        return self.peer_base.value + (parity & 1) * self.recv_bytes

    def copy(self, dst: int, src: int, nbytes: int, stream) -> None:
        raise_for_status(self.L.gp_copy_async(dst, src, nbytes, stream.cuda_stream), "gp_copy_async")

    def signal_sent(self, stream) -> None:
        raise_for_status(self.L.gp_event_record(self.sent, stream.cuda_stream), "gp_event_record")

    def wait_sent(self, stream) -> None:
        raise_for_status(self.L.gp_stream_wait_event(stream.cuda_stream, self.prev_sent), "gp_stream_wait_event")

    def signal_consumed(self, stream) -> None:
        raise_for_status(self.L.gp_event_record(self.consumed, stream.cuda_stream), "gp_event_record")

    def wait_consumed(self, stream) -> None:
        raise_for_status(self.L.gp_stream_wait_event(stream.cuda_stream, self.next_consumed),
                         "gp_stream_wait_event")

    # ---- per-frame hand-off (optional): one interprocess event per frame and
    # buffer parity, recorded after that frame's copy, so the successor can
    # decompress each frame as soon as it lands instead of after the last one.
    # Records and waits are "external", i.e. real event nodes inside captured
    # CUDA graphs.
    def enable_frame_events(self, nframes: int, cpu_group=None) -> None:
        L = self.L
        with torch.cuda.device(self.device):
            self.frame_sent = [[ctypes.c_void_p() for _ in range(nframes)] for _ in range(2)]
            handles = []
            for par in range(2):
                for i in range(nframes):
                    h = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
                    raise_for_status(L.gp_ipc_event_create(ctypes.byref(self.frame_sent[par][i]), h),
                                     "gp_ipc_event_create")
                    handles.append(bytes(h))
            objs = [None] * self.world
            dist.all_gather_object(objs, handles, group=cpu_group)
            prv = (self.rank - 1) % self.world
            self.prev_frame_sent = [[ctypes.c_void_p() for _ in range(nframes)] for _ in range(2)]
            for par in range(2):
                for i in range(nframes):
                    raise_for_status(L.gp_ipc_open_event(_handle(objs[prv][par * nframes + i]),
                                                         ctypes.byref(self.prev_frame_sent[par][i])),
                                     "gp_ipc_open_event")

    def signal_frame_sent(self, parity: int, i: int, stream) -> None:
        raise_for_status(self.L.gp_event_record_external(self.frame_sent[parity & 1][i], stream.cuda_stream),
                         "gp_event_record_external")

    def wait_frame_sent(self, parity: int, i: int, stream) -> None:
        raise_for_status(self.L.gp_stream_wait_event_external(stream.cuda_stream,
                                                              self.prev_frame_sent[parity & 1][i]),
                         "gp_stream_wait_event_external")

    def close(self) -> None:
        L = self.L
        for lst in getattr(self, "frame_sent", []) + getattr(self, "prev_frame_sent", []):
            for ev in lst:
                if ev.value:
                    L.gp_event_destroy(ev)
        self.frame_sent, self.prev_frame_sent = [], []
        if self.peer_base.value:
            L.gp_ipc_close_mem(self.peer_base)
            self.peer_base = ctypes.c_void_p()
        for ev in (self.sent, self.consumed, self.prev_sent, self.next_consumed):
            if ev.value:
                L.gp_event_destroy(ev)
        self.sent = self.consumed = self.prev_sent = self.next_consumed = ctypes.c_void_p()
        if self.recv_base.value:
            L.gp_peer_free(self.recv_base)
            self.recv_base = ctypes.c_void_p()


__all__ = ["PeerRing"]
