"""B200-native AdaTopK hot path of FusionLLM (arXiv 2410.12707).

Drop-in for the reference's `geopipe.compressor` (pkg/src/geopipe/compressor.py)
backed by hand-written sm_100a kernels behind a C-ABI (include/adatopk.h), plus
the compressed stage-boundary send/recv over NCCL (`transport`).
"""
from .compressor import (  # noqa: F401
    INDEX_BYTES,
    SPARSE_EXPANSION,
    VALUE_BYTES,
    CompressionPlan,
    SparsePayload,
    adatopk_plan,
    adatopk_plan_device,
    per_device_ratios,
    select_k,
    topk_compress,
    topk_decompress,
    uniform_plan,
    wire_bytes,
)
from .errors import EmptyVector, GeopipeError, IndexOutOfRange, InvalidRatio, NoCommunication  # noqa: F401

__version__ = "0.1.0"
