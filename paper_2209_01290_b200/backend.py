"""Kernel backend (reference pkg/src/nttmul/backend.py).

The reference chooses between its Cython kernels and a pure-Python twin.
This package has exactly one backend - the sm_100a CUDA library - and no
fallback: ``kernels()`` returns the :mod:`.kernels` surface, whose calls
raise if the library or the GPU is missing.  The selection functions keep
their names and error behaviour so callers written against the reference
keep working; asking for the CPU twin is an error.
"""

from __future__ import annotations

import os

from . import _lib
from . import kernels as _cuda

NAME = "native"  # the reference's name for the compiled backend
ALIASES = ("native", "cuda")


def native_available() -> bool:
    """True when the CUDA library loads (a GPU is needed to run it)."""
    try:
        _lib.load()
    except (ImportError, OSError):
        return False
    return True


def set_backend(name: str) -> None:
    """'native' / 'cuda' / 'auto' select the CUDA kernels; anything else is rejected."""
    if name == "auto" or name in ALIASES:
        if not native_available():
            raise RuntimeError("CUDA kernels are not available (library not built)")
        return
    if name == "python":
        raise RuntimeError("no CPU fallback: the pure-Python twin is not part of this "
                           "framework (use oracle/ for CPU checking)")
    raise ValueError(f"unknown backend {name!r}")


def active() -> str:
    return NAME


def kernels():
    """The active kernel module (always the CUDA surface)."""
    return _cuda


def get(name: str):
    if name in ALIASES:
        return _cuda
    if name == "python":
        raise RuntimeError("no CPU fallback in this framework")
    raise ValueError(f"unknown backend {name!r}")


_env = os.environ.get("NTTMUL_BACKEND")
if _env not in (None, "", "native", "cuda", "auto"):
    raise RuntimeError(f"NTTMUL_BACKEND={_env!r}: only the CUDA backend exists")
