"""Modular-reduction entry points (reference pkg/src/nttmul/modarith.py).

Two levels:

* Host constants and scalar reference semantics.  ``Modulus`` derives the
  per-prime constants of the paper's reductions (Alg. 2 classical, Alg. 3
  Dhem-Quisquater, Alg. 4 proposed) exactly as the reference does
  (modarith.py:34-83); the scalar functions keep the reference's argument
  order, assertions and ``ReductionStats`` bookkeeping.  They are host
  arithmetic on Python ints - what the plan layer uses to build constants -
  not the hot path.
* The hot path: :func:`mulmod` / :func:`barrett_proposed` & co. also accept
  CUDA uint64 tensors, in which case the element-wise product runs in the
  sm_100a Barrett kernel (``nttmul_hadamard``) with the chosen variant.

Variant table (mode, mu, s_in, s_out), m = bit length of q:
  builtin    (0, 0,               0,     0)      x % q
  classical  (1, 2^(2m)   // q,   m - 1, m + 1)  <= 2 corrections
  dhem       (2, 2^(2m+3) // q,   m - 2, m + 5)  <= 1 correction, m <= 60
  proposed   (2, 2^(2m+1) // q,   m - 2, m + 3)  <= 1 correction, m <= 62
"""

from __future__ import annotations

from dataclasses import dataclass, field

WORD_SIZE = 64

RED_BUILTIN = 0
RED_TWO_SUB = 1
RED_ONE_SUB = 2

VARIANTS = ("builtin", "classical", "dhem", "proposed")

# variant -> (mode, numerator exponent offset k in mu = 2^(2m+k)//q,
#             s_in offset, s_out offset)
_VARIANT_SHAPE = {
    "classical": (RED_TWO_SUB, 0, -1, +1),
    "dhem": (RED_ONE_SUB, 3, -2, +5),
    "proposed": (RED_ONE_SUB, 1, -2, +3),
}


class ModulusTooLargeError(ValueError):
    """The modulus is too wide for the requested reduction variant."""


def bit_length(a: int) -> int:
    """Bit length of a positive integer (paper §II <a>)."""
    if a < 1:
        raise ValueError(f"bit_length requires a >= 1, got {a}")
    return a.bit_length()


@dataclass(frozen=True)
class Modulus:
    """Odd modulus q (3 <= q < 2^62) and its reduction constants."""

    q: int
    m: int = field(init=False)
    mu_classical: int = field(init=False)
    mu_dhem: int | None = field(init=False)
    mu_proposed: int = field(init=False)
    half_q_ceil: int = field(init=False)

    def __post_init__(self):
        q = self.q
        if q < 3 or q % 2 == 0:
            raise ValueError(f"modulus must be odd and >= 3, got {q}")
        m = q.bit_length()
        if m > WORD_SIZE - 2:
            raise ModulusTooLargeError(
                f"modulus has {m} bits; at most {WORD_SIZE - 2} supported")
        put = object.__setattr__
        put(self, "m", m)
        put(self, "mu_classical", (1 << 2 * m) // q)
        put(self, "mu_dhem", (1 << 2 * m + 3) // q if m <= WORD_SIZE - 4 else None)
        put(self, "mu_proposed", (1 << 2 * m + 1) // q)
        put(self, "half_q_ceil", (q + 1) // 2)

    def reduction_params(self, variant: str) -> tuple[int, int, int, int]:
        """(mode, mu, shift_in, shift_out) for a variant (modarith.py:68-83)."""
        if variant == "builtin":
            return RED_BUILTIN, 0, 0, 0
        shape = _VARIANT_SHAPE.get(variant)
        if shape is None:
            raise ValueError(f"unknown reduction variant {variant!r}")
        mode, k, di, do = shape
        if variant == "dhem" and self.mu_dhem is None:
            raise ModulusTooLargeError(
                f"dhem variant requires m <= {WORD_SIZE - 4}, got m={self.m}")
        mu = {"classical": self.mu_classical, "dhem": self.mu_dhem,
              "proposed": self.mu_proposed}[variant]
        assert mu == (1 << 2 * self.m + k) // self.q
        return mode, mu, self.m + di, self.m + do


@dataclass
class ReductionStats:
    """How many reductions needed 0, 1 or >= 2 correctional subtractions."""

    calls: int = 0
    subtractions_0: int = 0
    subtractions_1: int = 0
    subtractions_2: int = 0

    def record(self, nsubs: int) -> None:
        self.calls += 1
        slot = min(nsubs, 2)
        name = f"subtractions_{slot}"
        setattr(self, name, getattr(self, name) + 1)

    def merge(self, other: "ReductionStats") -> None:
        for name in ("calls", "subtractions_0", "subtractions_1", "subtractions_2"):
            setattr(self, name, getattr(self, name) + getattr(other, name))


def mod_add(a: int, b: int, mod: Modulus) -> int:
    """(a + b) mod q, one conditional subtraction (paper Alg. 1)."""
    assert 0 <= a < mod.q and 0 <= b < mod.q, "inputs must be reduced"
    s = a + b
    return s - mod.q if s >= mod.q else s


def mod_sub(a: int, b: int, mod: Modulus) -> int:
    """(a - b) mod q, one conditional addition."""
    assert 0 <= a < mod.q and 0 <= b < mod.q, "inputs must be reduced"
    d = a - b
    return d + mod.q if d < 0 else d


def reduce_builtin(x: int, q: int) -> int:
    """x mod q by division - the oracle every variant must agree with."""
    if q < 1:
        raise ValueError(f"modulus must be >= 1, got {q}")
    return x % q


def half_mod(x: int, mod: Modulus) -> int:
    """x / 2 mod q as (x >> 1) + (x & 1) * (q + 1)/2 (no division)."""
    assert 0 <= x < mod.q, "input must be reduced"
    return (x >> 1) + (x & 1) * mod.half_q_ceil


def _barrett_scalar(x: int, mod: Modulus, variant: str,
                    stats: ReductionStats | None) -> int:
    _, mu, s_in, s_out = mod.reduction_params(variant)
    assert 0 <= x < (1 << 2 * mod.m), "operand exceeds 2^(2m)"
    r = x - ((((x >> s_in) * mu) >> s_out) * mod.q)
    k = 0
    while r >= mod.q:
        r -= mod.q
        k += 1
    if stats is not None:
        stats.record(k)
    return r


def _tensor_mulmod(a, b, mod: Modulus, variant: str):
    """Element-wise a*b mod q on the GPU with the given variant."""
    from . import kernels  # local: keeps host constants importable without CUDA

    return kernels.mulmod_tensor(a, b, mod, variant)


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def barrett_classical(x, mod: Modulus, stats: ReductionStats | None = None):
    """Classical Barrett (Alg. 2): up to two correctional subtractions."""
    return _barrett_scalar(x, mod, "classical", stats)


def barrett_dhem(x, mod: Modulus, stats: ReductionStats | None = None):
    """Dhem-Quisquater (Alg. 3): one correction, m <= 60."""
    return _barrett_scalar(x, mod, "dhem", stats)


def barrett_proposed(x, mod: Modulus, stats: ReductionStats | None = None):
    """The paper's variant (Alg. 4): one correction, m <= 62."""
    return _barrett_scalar(x, mod, "proposed", stats)


def mulmod(a, b, mod: Modulus, variant: str = "proposed",
           stats: ReductionStats | None = None):
    """a * b mod q with the selected reduction.

    Python ints: scalar reference semantics (modarith.py:169-178).
    CUDA uint64 tensors (same shape): the sm_100a Barrett kernel, returning a
    new tensor; ``stats`` is not tracked on the device path.
    """
    if _is_tensor(a) or _is_tensor(b):
        return _tensor_mulmod(a, b, mod, variant)
    assert 0 <= a < mod.q and 0 <= b < mod.q, "inputs must be reduced"
    if variant == "builtin":
        if stats is not None:
            stats.record(0)
        return (a * b) % mod.q
    return _barrett_scalar(a * b, mod, variant, stats)
