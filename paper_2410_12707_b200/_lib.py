"""ctypes binding of libadatopk.so (the C-ABI in include/adatopk.h).

There is no CPU fallback: if the library is missing the import of any compute
entry point fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int32, c_int64, c_size_t, c_void_p, POINTER
from pathlib import Path

LIB_PATH = Path(os.environ.get("GP_LIB") or Path(__file__).resolve().parent / "_lib" / "libadatopk.so")

DTYPE_F32 = 0
DTYPE_BF16 = 1
DTYPE_F64 = 2
FLAG_OUT_OF_RANGE = 1
FLAG_UNSORTED = 2
FLAG_HEADER = 4   # frame header {d, k} disagrees with the receiver's expectation
FLAG_BAD_K = 8    # device-resident k outside [1, min(k_cap, d)]
FLAG_ENVELOPE = 16  # a message's OpData envelope differs from the receiver's expectation
ENVELOPE_WORDS = 16
ENVELOPE_BYTES = 128
FRAME_HEADER_BYTES = 16

_SIGS = {
    "gp_version": (ctypes.c_char_p, []),
    "gp_select_k": (c_int, [c_int64, c_double, POINTER(c_int64)]),
    "gp_set_cluster_path": (c_int, [c_int]),
    "gp_wire_bytes": (c_int, [c_int64, c_double, POINTER(c_int64)]),
    "gp_topk_workspace_bytes": (c_size_t, [c_int64, c_int]),
    "gp_workspace_init": (c_int, [c_void_p, c_size_t, c_void_p]),
    "gp_topk_compress": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int, c_void_p, c_int,
                                 c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "gp_topk_compress_frame": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_void_p, c_size_t,
                                       c_void_p]),
    "gp_topk_compress_ctas": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int, c_void_p, c_int,
                                      c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_int]),
    "gp_topk_compress_frame_ctas": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_void_p, c_size_t,
                                            c_void_p, c_int]),
    "gp_topk_decompress": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int64, c_int64, c_void_p, c_int, c_int,
                                   c_void_p, c_void_p]),
    "gp_topk_decompress_frame": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int, c_int, c_void_p,
                                         c_void_p]),
    "gp_topk_compress_frame_dk": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                          c_size_t, c_void_p, c_int]),
    "gp_topk_decompress_frame_dk": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int, c_int, c_void_p,
                                            c_void_p]),
    "gp_pack_frame": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int64, c_int64, c_void_p, c_void_p]),
    "gp_envelope_write": (c_int, [c_void_p, POINTER(c_int64), c_void_p]),
    "gp_envelope_check": (c_int, [c_void_p, POINTER(c_int64), ctypes.c_uint64, c_void_p, c_void_p]),
    "gp_unpack_frame": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                c_void_p]),
    "gp_topk_decompress_unsorted": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int64, c_int64, c_void_p, c_int,
                                            c_void_p, c_void_p, c_void_p]),
    "gp_adatopk_plan": (c_int, [POINTER(c_double), c_int, c_double, POINTER(c_int64), POINTER(c_double),
                                POINTER(c_int64), POINTER(c_int32), c_void_p]),
    "gp_adatopk_plan_host": (c_int, [POINTER(c_double), c_int, c_double, POINTER(c_int64), POINTER(c_double),
                                     POINTER(c_int64)]),
    # peer-memory transport (include/adatopk.h)
    "gp_peer_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "gp_peer_free": (c_int, [c_void_p]),
    "gp_ipc_mem_handle": (c_int, [c_void_p, c_void_p]),
    "gp_ipc_open_mem": (c_int, [c_void_p, POINTER(c_void_p)]),
    "gp_ipc_close_mem": (c_int, [c_void_p]),
    "gp_ipc_event_create": (c_int, [POINTER(c_void_p), c_void_p]),
    "gp_ipc_open_event": (c_int, [c_void_p, POINTER(c_void_p)]),
    "gp_event_destroy": (c_int, [c_void_p]),
    "gp_event_record": (c_int, [c_void_p, c_void_p]),
    "gp_stream_wait_event": (c_int, [c_void_p, c_void_p]),
    "gp_event_record_external": (c_int, [c_void_p, c_void_p]),
    "gp_stream_wait_event_external": (c_int, [c_void_p, c_void_p]),
    "gp_copy_async": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
}
IPC_HANDLE_BYTES = 64

EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the AdaTopK path has no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
