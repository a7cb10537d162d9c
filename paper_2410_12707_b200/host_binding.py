"""NumPy-facing binding of the GPU compressor for the reference's host executor.

The reference executor (pkg/src/geopipe/executor.py:16,207-220) keeps every
tensor in NumPy:

    sp = topk_compress(np.asarray(payload).reshape(-1), ratio)   # :213
    ...
    return topk_decompress(payload).reshape(shape)                # :220

and does NumPy arithmetic on what `topk_decompress` returns.  The drop-in
`paper_2410_12707_b200.topk_decompress` returns a CUDA tensor, so binding it by
name alone would break the next NumPy op.  This module's two functions run
the same sm_100a kernels (the input is copied to the current CUDA device and
the payload stays in HBM), and `topk_decompress` copies the dense result back
into a NumPy array of the payload's dtype (float64 for the executor's
tensors; the f64 key path keeps the selection exact).

    import geopipe.executor as ex, geopipe.errors as er
    from paper_2410_12707_b200 import host_binding
    undo = host_binding.patch_executor(ex, er)   # the executor now compresses on the GPU
    ...
    undo()

With the reference's errors module given, the four compressor exceptions are
re-raised as the reference's own classes (errors.py:46-59), so callers that
catch them keep working.
"""
from __future__ import annotations

import functools

import numpy as np

from . import compressor as _c
from . import errors as _e

_NAMES = ("InvalidRatio", "EmptyVector", "IndexOutOfRange", "NoCommunication")


def _translate(errors_module):
    def deco(fn):
        if errors_module is None:
            return fn

        @functools.wraps(fn)
        def wrapped(*a, **kw):
            try:
                return fn(*a, **kw)
            except _e.GeopipeError as exc:
                for name in _NAMES:
                    if isinstance(exc, getattr(_e, name)):
                        raise getattr(errors_module, name)(*exc.args) from exc
                raise

        return wrapped

    return deco


def topk_compress(vector, ratio: float) -> _c.SparsePayload:
    """compressor.py:79-94 on the GPU; the payload's tensors stay on the device."""
    return _c.topk_compress(vector, ratio)


def topk_decompress(payload) -> np.ndarray:
    """compressor.py:97-103 on the GPU; returns a NumPy array of the values' dtype."""
    return _c.topk_decompress(payload).cpu().numpy()


def patch_executor(executor_module, errors_module=None):
    """Rebind `topk_compress` / `topk_decompress` in `executor_module` (the names
    executor.py:16 imports).  Returns a callable that restores the originals."""
    old = (executor_module.topk_compress, executor_module.topk_decompress)
    executor_module.topk_compress = _translate(errors_module)(topk_compress)
    executor_module.topk_decompress = _translate(errors_module)(topk_decompress)

    def undo():
        executor_module.topk_compress, executor_module.topk_decompress = old

    return undo


__all__ = ["topk_compress", "topk_decompress", "patch_executor"]
