"""CPU oracle for the polymul hot path - TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / CPU baseline; the product package
``paper_2209_01290_b200`` never imports it and fails loudly without its CUDA
library.

Two checkers live here:

* ``ntt_oracle.c`` (built to ``libntt_oracle.so`` by :func:`build`) - a plain-C
  restatement of the reference kernel core
  (/root/reference/pkg/src/nttmul/_kernels.pyx), each function citing the
  reference lines it follows.  Pinned against the reference's own outputs by
  ``tests/test_oracle.py`` and the golden vectors in ``tests/golden/``.
* ``_ref/`` - the UNMODIFIED reference package (``nttmul`` with its Cython
  backend) built by ``build_ref.sh`` from /root/reference (git-ignored; it
  travels to the GPU box with the repo snapshot).  :func:`reference` imports it
  when present.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libntt_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_lib = None


def build(force: bool = False) -> str:
    """Compile ntt_oracle.c with gcc (seconds)."""
    src = os.path.join(HERE, "ntt_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", LIB, src])
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        i64, u64, c_int = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        L.oracle_ntt_ct.argtypes = [_u64p, i64, _u64p, u64, c_int, u64, c_int, c_int, c_int, _u64p]
        L.oracle_intt_gs.argtypes = [_u64p, i64, _u64p, u64, u64, c_int, u64, c_int, c_int,
                                     c_int, c_int, _u64p]
        L.oracle_fused_middle.argtypes = [_u64p, _u64p, _u64p, i64, _u64p, u64, c_int, u64,
                                          c_int, c_int, _u64p]
        L.oracle_hadamard.argtypes = [_u64p, _u64p, _u64p, i64, u64, c_int, u64, c_int, c_int,
                                      _u64p]
        L.oracle_scale.argtypes = [_u64p, i64, u64, u64, c_int, u64, c_int, c_int, _u64p]
        L.oracle_negacyclic_naive.argtypes = [_u64p, _u64p, _u64p, i64, u64, _u64p]
        L.oracle_mulmod_loop.argtypes = [_u64p, _u64p, i64, u64, c_int, u64, c_int, c_int, u64]
        L.oracle_mulmod_loop.restype = u64
        L.oracle_polymul_fused.argtypes = [_u64p, _u64p, _u64p, i64, _u64p, _u64p, u64, c_int,
                                           u64, c_int, c_int, _u64p, _u64p]
        L.oracle_twiddles.argtypes = [u64, u64, u64, c_int, _u64p, _u64p]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def _arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


# ---- reduction parameters (restates modarith.py:49-83) -------------------

def reduction_params(q: int, variant: str = "proposed"):
    """(mode, mu, s_in, s_out) exactly as Modulus.reduction_params."""
    m = q.bit_length()
    if variant == "builtin":
        return 0, 0, 0, 0
    if variant == "classical":
        return 1, (1 << (2 * m)) // q, m - 1, m + 1
    if variant == "dhem":
        if m > 60:
            raise ValueError("dhem needs m <= 60")
        return 2, (1 << (2 * m + 3)) // q, m - 2, m + 5
    if variant == "proposed":
        return 2, (1 << (2 * m + 1)) // q, m - 2, m + 3
    raise ValueError(variant)


def twiddles(q: int, psi: int, log_n: int):
    """(tw_fwd, tw_inv) as params._plan_from_root builds them."""
    n = 1 << log_n
    f = np.empty(n, dtype=np.uint64)
    v = np.empty(n, dtype=np.uint64)
    lib().oracle_twiddles(q, psi, pow(psi, q - 2, q), log_n, _p(f), _p(v))
    return f, v


# ---- kernel surface (same argument order as the reference _kernels) ------

def ntt_ct(a, tw, q, mode, mu, s_in, s_out, truncate, counts=None):
    lib().oracle_ntt_ct(_p(a), len(a), _p(tw), q, mode, mu, s_in, s_out, int(truncate),
                        _p(counts))


def intt_gs(a, tw, q, half_q, mode, mu, s_in, s_out, scaled, skip_first, counts=None):
    lib().oracle_intt_gs(_p(a), len(a), _p(tw), q, half_q, mode, mu, s_in, s_out,
                         int(scaled), int(skip_first), _p(counts))


def fused_middle(ah, bh, ch, tw, q, mode, mu, s_in, s_out, counts=None):
    lib().oracle_fused_middle(_p(ah), _p(bh), _p(ch), len(ah), _p(tw), q, mode, mu, s_in,
                              s_out, _p(counts))


def hadamard(a, b, out, q, mode, mu, s_in, s_out, counts=None):
    lib().oracle_hadamard(_p(a), _p(b), _p(out), len(a), q, mode, mu, s_in, s_out, _p(counts))


def scale(a, factor, q, mode, mu, s_in, s_out, counts=None):
    lib().oracle_scale(_p(a), len(a), factor, q, mode, mu, s_in, s_out, _p(counts))


def negacyclic_naive(a, b, q, counts=None) -> np.ndarray:
    a, b = _arr(a), _arr(b)
    out = np.empty(len(a), dtype=np.uint64)
    lib().oracle_negacyclic_naive(_p(a), _p(b), _p(out), len(a), q, _p(counts))
    return out


def mulmod_loop(a, b, q, mode, mu, s_in, s_out, passes) -> int:
    a, b = _arr(a), _arr(b)
    return int(lib().oracle_mulmod_loop(_p(a), _p(b), len(a), q, mode, mu, s_in, s_out,
                                        passes))


def polymul_fused(a, b, q: int, psi: int, variant: str = "proposed", counts=None,
                  tables=None) -> np.ndarray:
    """Reference polymul_fused for one prime, from (q, psi)."""
    a, b = _arr(a), _arr(b)
    n = len(a)
    log_n = n.bit_length() - 1
    tw_f, tw_i = tables if tables is not None else twiddles(q, psi, log_n)
    mode, mu, s_in, s_out = reduction_params(q, variant)
    c = np.empty(n, dtype=np.uint64)
    scratch = np.empty(2 * n, dtype=np.uint64)
    lib().oracle_polymul_fused(_p(a), _p(b), _p(c), n, _p(tw_f), _p(tw_i), q, mode, mu,
                               s_in, s_out, _p(scratch), _p(counts))
    return c


def polymul_rns(a: np.ndarray, b: np.ndarray, primes, psis, variant="proposed",
                tables=None) -> np.ndarray:
    """[B, L, n] batched fused polymul (rns.py:116-119 per ciphertext)."""
    a, b = _arr(a), _arr(b)
    B, L, n = a.shape
    log_n = n.bit_length() - 1
    out = np.empty_like(a)
    if tables is None:
        tables = [twiddles(q, psi, log_n) for q, psi in zip(primes, psis)]
    for bi in range(B):
        for li, q in enumerate(primes):
            out[bi, li] = polymul_fused(a[bi, li], b[bi, li], q, 0, variant,
                                        tables=tables[li])
    return out


# ---- RNS / CRT (reference rns.py:82-108), Python big integers -------------

def crt_decompose(values, primes) -> np.ndarray:
    """residues[i, j] = values[j] mod primes[i] (rns.py:82-91)."""
    vals = [int(v) for v in values]
    return np.array([[v % q for v in vals] for q in primes], dtype=np.uint64).reshape(
        len(primes), len(vals))


def crt_reconstruct(residues, primes) -> list[int]:
    """The unique vector in [0, prod q) with the given residues (rns.py:94-108)."""
    big_q = 1
    for q in primes:
        big_q *= int(q)
    weights = [(big_q // int(q), pow(big_q // int(q) % int(q), -1, int(q))) for q in primes]
    rows = [[int(x) for x in r] for r in residues]
    out = []
    for j in range(len(rows[0])):
        acc = 0
        for r, q, (quot, inv) in zip(rows, primes, weights):
            acc += r[j] * inv % int(q) * quot
        out.append(acc % big_q)
    return out


# ---- the unmodified reference (oracle/_ref) -------------------------------

def reference():
    """Import the reference package built into oracle/_ref (or None)."""
    if not os.path.isdir(os.path.join(REF_DIR, "nttmul")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import nttmul  # noqa: PLC0415

    return nttmul
