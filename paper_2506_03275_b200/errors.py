"""Exception classes mirroring the reference's ``csd::Error`` hierarchy
(/root/reference/proj/include/csd/error.hpp:8-46) and the C-ABI status mapping."""
from __future__ import annotations

import builtins


class Error(RuntimeError):
    """csd::Error"""


class ShapeError(Error):
    """Shape disagreement, including chunk-divisibility violations."""


class IndexError(Error, builtins.IndexError):  # noqa: A001 - mirrors csd::IndexError
    """An index outside its valid range or duplicated."""


class NumericError(Error):
    """Non-finite input."""


class StateError(Error):
    """Sparse step before any dense step."""


class ValueError(Error, builtins.ValueError):  # noqa: A001 - mirrors csd::ValueError
    """Parameter outside its documented range (e.g. top-k count)."""


class ConfigError(Error):
    """Invalid model / voxel configuration."""


class CudaError(Error):
    """CUDA runtime or launch failure."""


class UnsupportedError(Error):
    """Shape outside the production kernel envelope (no fallback exists)."""


_BY_STATUS = {1: ShapeError, 2: IndexError, 3: NumericError, 4: StateError, 5: ValueError,
              6: ConfigError, 7: CudaError, 8: UnsupportedError}


def raise_for(lib, status: int) -> None:
    if status == 0:
        return
    msg = lib.csd_last_error()
    msg = msg.decode() if msg else ""
    raise _BY_STATUS.get(status, Error)(msg or f"csd status {status}")
