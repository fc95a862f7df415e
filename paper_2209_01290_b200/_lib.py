"""ctypes binding of the C ABI in include/nttmul_b200.h.

This is the Python-side "FFI stub" of the drop-in boundary: the reference's
Cython module boundary (_kernels.pyx) is replaced by a plain C ABI over device
pointers, and this module binds it.  There is no fallback: if the CUDA library
is missing or no GPU is present, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libnttmul_b200.so"
# NTTMUL_LIB: an alternative build of the same ABI (A/B measurements only)
LIB_PATH = os.environ.get("NTTMUL_LIB") or os.path.join(HERE, LIB_NAME)

ABI_VERSION = 1
SCHED_AUTO, SCHED_THREE, SCHED_CLUSTER, SCHED_PASSES, SCHED_GRID = 0, 1, 2, 3, 4

_c_u64 = ctypes.c_uint64
_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_vp = ctypes.c_void_p


class NttmulError(RuntimeError):
    """A non-zero status returned by the CUDA library."""


class LimbStruct(ctypes.Structure):
    """Mirror of nttmul_limb_t (96 bytes)."""

    _fields_ = [
        ("q", _c_u64),
        ("mu_sh", _c_u64),
        ("sc_full", _c_u64 * 4),
        ("sc_skip", _c_u64 * 4),
        ("s_in", ctypes.c_uint32),
        ("s_hi", ctypes.c_uint32),
        ("mode", ctypes.c_uint32),
        ("log_n", ctypes.c_uint32),
    ]


assert ctypes.sizeof(LimbStruct) == 96

# name -> (restype, argtypes)
_PROTOS = {
    "nttmul_abi_version": (_c_int, []),
    "nttmul_last_error": (ctypes.c_char_p, []),
    "nttmul_limb_prepare": (_c_int, [ctypes.POINTER(LimbStruct), _c_u64, _c_int, _c_u64,
                                     _c_int, _c_int, _c_int, _c_u64]),
    "nttmul_twiddle_tables": (_c_int, [_vp, _vp, _vp, _vp, _c_u64, _c_u64, _c_u64, _c_int,
                                       _vp]),
    "nttmul_shoup_pairs": (_c_int, [_vp, _vp, _c_u64, _c_i64, _vp]),
    "nttmul_check_twiddles": (_c_int, [_vp, _vp, _c_u64, _c_i64, _vp, _vp]),
    "nttmul_ntt_ct": (_c_int, [_vp, _vp, _c_u64, _c_int, _c_u64, _c_int, _c_int, _c_int,
                               _c_int, _c_i64, _vp]),
    "nttmul_intt_gs": (_c_int, [_vp, _vp, _c_u64, _c_u64, _c_int, _c_u64, _c_int, _c_int,
                                _c_int, _c_int, _c_int, _c_i64, _c_u64, _vp]),
    "nttmul_fused_middle": (_c_int, [_vp, _vp, _vp, _vp, _c_u64, _c_int, _c_u64, _c_int,
                                     _c_int, _c_int, _c_i64, _vp]),
    "nttmul_hadamard": (_c_int, [_vp, _vp, _vp, _c_i64, _c_u64, _c_int, _c_u64, _c_int,
                                 _c_int, _vp]),
    "nttmul_scale": (_c_int, [_vp, _c_u64, _c_i64, _c_u64, _c_int, _c_u64, _c_int, _c_int,
                              _vp]),
    "nttmul_mulmod_loop": (_c_int, [_vp, _vp, _c_i64, _c_u64, _c_int, _c_u64, _c_int,
                                    _c_int, _c_u64, _vp, _vp]),
    "nttmul_polymul_fused_rns": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                          _c_i64, _c_int, _vp, _vp]),
    "nttmul_set_schedule": (_c_int, [_c_int, _c_int, _c_int]),
    "nttmul_set_split": (_c_int, [_c_int, _c_int]),
    "nttmul_polymul_fused_rns_phases": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                                 _c_i64, _c_int, _vp, _c_int, _vp]),
    "nttmul_polymul_fused_rns_host": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                               _c_i64, _c_int, _vp, _c_i64, _vp]),
    "nttmul_negacyclic_naive": (_c_int, [_vp, _vp, _vp, _c_u64, _c_i64, _c_i64, _vp]),
    "nttmul_sweep_random": (_c_int, [_c_int, _c_u64, _c_u64, _vp, _vp, _vp]),
    "nttmul_sweep_exhaustive": (_c_int, [_c_u64, _c_u64, _vp, _vp, _vp]),
    "nttmul_gather": (_c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _vp]),
    "nttmul_crt_decompose": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_i64, _c_i64, _vp]),
    "nttmul_crt_reconstruct": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                        _c_i64, _c_i64, _vp]),
    "nttmul_modmul_roof": (_c_int, [ctypes.POINTER(LimbStruct), _c_int, _c_int, _c_int,
                                    _c_i64, _vp, ctypes.POINTER(ctypes.c_double), _vp]),
}

EXPORTED = tuple(_PROTOS)

HOST_NBUF = 3  # NTTMUL_HOST_NBUF

_lib = None


def load(path: str | None = None):
    """Load (once) and return the CUDA library; raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("NTTMUL_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{LIB_NAME} not built at {p}: run `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(p)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.nttmul_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_NAME}: ABI {lib.nttmul_abi_version()} != {ABI_VERSION}")
    if path is None:
        _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().nttmul_last_error().decode(errors="replace")
        raise NttmulError(f"{what}: status {status}: {msg}")


def call(name: str, *args) -> None:
    """Invoke an entry point and raise NttmulError on a non-zero status."""
    check(getattr(load(), name)(*args), name)


def prepare_limb(q: int, mode: int, mu: int, s_in: int, s_out: int, log_n: int,
                 w1_inv: int) -> LimbStruct:
    limb = LimbStruct()
    call("nttmul_limb_prepare", ctypes.byref(limb), q, mode, mu, s_in, s_out, log_n, w1_inv)
    return limb
