"""Error hierarchy mirroring epikv (numerics.hpp:21-34, kvcache.hpp:22-25).

C-ABI status codes (include/epk/epk.h) map back onto the same classes the
reference throws, with the reference's message prefixes where it has them.
"""


class Error(RuntimeError):
    """epikv::Error."""


class DimensionError(Error):
    """epikv::DimensionError."""


class ZeroNormError(Error):
    """epikv::ZeroNormError."""


class IoError(Error):
    """epikv::IoError."""


class CudaError(Error):
    """A CUDA runtime failure below the C ABI (no reference counterpart)."""


class UnsupportedError(Error):
    """A shape outside what the sm_100a kernels support."""


def raise_for_status(rc: int, msg: str) -> None:
    if rc == -3:
        raise DimensionError(msg)
    if rc == -4:
        raise ZeroNormError(msg)
    if rc == -7:
        raise CudaError(msg)
    if rc == -8:
        raise UnsupportedError(msg)
    raise Error(msg or f"epk status {rc}")
