"""Exception types of the compressor boundary.

Names and hierarchy mirror the reference's shared error module
(/root/reference/pkg/src/geopipe/errors.py:4-59) for the four classes the
compressor raises, so callers written against `geopipe.compressor` catch the
same names.  The C-ABI status codes (include/adatopk.h) map onto them 1:1.
"""


class GeopipeError(Exception):
    """Base class (errors.py:4-5)."""


class InvalidRatio(GeopipeError):
    """ratio < 1 (errors.py:46; raised at compressor.py:74-75, 118-119, 134-135)."""


class EmptyVector(GeopipeError):
    """d == 0 (errors.py:50; compressor.py:88-89)."""


class IndexOutOfRange(GeopipeError):
    """index < 0 or >= d on decompress (errors.py:54; compressor.py:99-100)."""


class NoCommunication(GeopipeError):
    """max link time <= 0 (errors.py:58; compressor.py:121-122)."""


GP_OK = 0
GP_ERR_INVALID_RATIO = 1
GP_ERR_EMPTY_VECTOR = 2
GP_ERR_INDEX_OUT_OF_RANGE = 3
GP_ERR_NO_COMMUNICATION = 4
GP_ERR_CUDA = 5
GP_ERR_INVALID_ARGUMENT = 6


def raise_for_status(status: int, what: str = "", payload=None) -> None:
    """Translate a C-ABI status code into the reference exception."""
    if status == GP_OK:
        return
    if status == GP_ERR_INVALID_RATIO:
        raise InvalidRatio(payload)
    if status == GP_ERR_EMPTY_VECTOR:
        raise EmptyVector("cannot compress a zero-length vector")
    if status == GP_ERR_INDEX_OUT_OF_RANGE:
        raise IndexOutOfRange(payload)
    if status == GP_ERR_NO_COMMUNICATION:
        raise NoCommunication("all link communication estimates are zero")
    if status == GP_ERR_CUDA:
        raise RuntimeError(f"CUDA error in {what}")
    raise ValueError(f"invalid argument to {what} (status {status})")
