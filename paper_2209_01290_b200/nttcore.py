"""Forward / inverse transforms on the GPU (reference pkg/src/nttmul/nttcore.py).

Public entry points keep the reference signatures - ``ntt_ct(a, plan, ctr)``
etc. take a :class:`Polynomial` and mutate it in place, re-tagging its
ordering - and dispatch through ``backend.kernels()`` exactly like the
reference (nttcore.py:102-185), so the kernel surface is the one boundary.
A Polynomial's coefficients live in HBM as a CUDA uint64 tensor.

Batching: the reference's ``batch_ntt`` fans rows out to a thread pool
(nttcore.py:503-533); here the rows are stacked into one [B, n] tensor and
transformed by ONE launch (the batch is the CUDA grid), then scattered back,
so the result is identical for any ``workers`` value by construction.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, backend
from .kernels import C_ADDSUB, C_HALF, C_MODMUL, C_NEG, C_TWIDDLE
from .params import NttPlan

NORMAL = "normal"
BIT_REVERSED = "bit_reversed"
TRUNCATED = "truncated"
VENDOR_2D = "vendor_2d"


@dataclass
class OpCounter:
    """Tallies of the arithmetic the reference algorithm performs."""

    modmul: int = 0
    modadd_sub: int = 0
    half_scalings: int = 0
    twiddle_loads: int = 0
    negations: int = 0

    def add_array(self, counts) -> None:
        self.modmul += int(counts[C_MODMUL])
        self.modadd_sub += int(counts[C_ADDSUB])
        self.half_scalings += int(counts[C_HALF])
        self.twiddle_loads += int(counts[C_TWIDDLE])
        self.negations += int(counts[C_NEG])

    def merge(self, other: "OpCounter") -> None:
        self.modmul += other.modmul
        self.modadd_sub += other.modadd_sub
        self.half_scalings += other.half_scalings
        self.twiddle_loads += other.twiddle_loads
        self.negations += other.negations

    def as_tuple(self) -> tuple[int, int, int, int, int]:
        return (self.modmul, self.modadd_sub, self.half_scalings, self.twiddle_loads,
                self.negations)


class Polynomial:
    """Length-n residue vector in HBM plus its ordering tag."""

    __slots__ = ("coeffs", "ordering")

    def __init__(self, coeffs, ordering: str = NORMAL):
        self.coeffs = _device.to_device(coeffs)
        self.ordering = ordering

    @classmethod
    def from_list(cls, values, ordering: str = NORMAL) -> "Polynomial":
        return cls(np.array([int(v) for v in values], dtype=np.uint64), ordering)

    @classmethod
    def random(cls, plan: NttPlan, rng) -> "Polynomial":
        """Same draw sequence as the reference (``rng.randrange(q)`` n times)."""
        return cls.from_list([rng.randrange(plan.q) for _ in range(plan.n)])

    @classmethod
    def unit(cls, n: int, index: int = 0) -> "Polynomial":
        c = np.zeros(n, dtype=np.uint64)
        c[index] = 1
        return cls(c)

    def copy(self) -> "Polynomial":
        return Polynomial(self.coeffs.clone(), self.ordering)

    def numpy(self) -> np.ndarray:
        return self.coeffs.cpu().numpy()

    def to_list(self) -> list[int]:
        return [int(x) for x in self.numpy()]

    def __len__(self) -> int:
        return int(self.coeffs.numel())

    def __repr__(self) -> str:
        return f"Polynomial(n={len(self)}, ordering={self.ordering!r})"


def _check(a: Polynomial, plan: NttPlan, ordering: str) -> None:
    if len(a) != plan.n:
        raise ValueError(f"length {len(a)} does not match plan n={plan.n}")
    if a.ordering != ordering:
        raise ValueError(f"expected {ordering}-order input, got {a.ordering}")


def _counts() -> np.ndarray:
    return np.zeros(5, dtype=np.uint64)


def _finish(ctr: OpCounter | None, counts: np.ndarray) -> None:
    if ctr is not None:
        ctr.add_array(counts)


def ntt_ct(a: Polynomial, plan: NttPlan, ctr: OpCounter | None = None) -> Polynomial:
    """Merged forward NTT in place: normal -> bit-reversed order."""
    _check(a, plan, NORMAL)
    counts = _counts()
    backend.kernels().ntt_ct(a.coeffs, plan.tw_fwd, *plan.red_args, False, counts)
    _finish(ctr, counts)
    a.ordering = BIT_REVERSED
    return a


def ntt_ct_truncated(a: Polynomial, plan: NttPlan,
                     ctr: OpCounter | None = None) -> Polynomial:
    """Forward NTT without its final stage (input of the fused middle)."""
    if plan.n < 4:
        raise ValueError("truncation needs n >= 4")
    _check(a, plan, NORMAL)
    counts = _counts()
    backend.kernels().ntt_ct(a.coeffs, plan.tw_fwd, *plan.red_args, True, counts)
    _finish(ctr, counts)
    a.ordering = TRUNCATED
    return a


def _inverse(a: Polynomial, plan: NttPlan, ctr, scaled: bool, skip: bool,
             ordering: str) -> Polynomial:
    _check(a, plan, ordering)
    q, mode, mu, s_in, s_out = plan.red_args
    counts = _counts()
    backend.kernels().intt_gs(a.coeffs, plan.tw_inv, q, plan.mod.half_q_ceil, mode, mu,
                              s_in, s_out, scaled, skip, counts)
    _finish(ctr, counts)
    a.ordering = NORMAL
    return a


def intt_gs(a: Polynomial, plan: NttPlan, ctr: OpCounter | None = None) -> Polynomial:
    """Merged inverse NTT without 1/n: the result is n times the inverse."""
    return _inverse(a, plan, ctr, False, False, BIT_REVERSED)


def intt_gs_scaled(a: Polynomial, plan: NttPlan,
                   ctr: OpCounter | None = None) -> Polynomial:
    """Merged inverse NTT including 1/n (folded into the last stage)."""
    return _inverse(a, plan, ctr, True, False, BIT_REVERSED)


def intt_gs_truncated(a: Polynomial, plan: NttPlan,
                      ctr: OpCounter | None = None) -> Polynomial:
    """Scaled inverse without its first stage (after the fused middle)."""
    if plan.n < 4:
        raise ValueError("truncation needs n >= 4")
    return _inverse(a, plan, ctr, True, True, TRUNCATED)


def scale_by(factor: int, a: Polynomial, plan: NttPlan,
             ctr: OpCounter | None = None) -> Polynomial:
    """a <- factor * a mod q, in place."""
    counts = _counts()
    backend.kernels().scale(a.coeffs, factor, *plan.red_args, counts)
    _finish(ctr, counts)
    return a


# ---------------------------------------------------------------------------
# radix-4 shapes (reference nttcore.py:189-329): two merged radix-2 stages per
# pass.  Their output order and values equal the radix-2 transforms exactly
# (the reference's own contract), and on the GPU every transform already runs
# several stages per register pass (radix-8 row passes, radix-16 column
# passes), so they execute the same kernels; only the bookkeeping is the
# radix-4 loop's.

def _radix4_counts(n: int, inverse: bool) -> np.ndarray:
    """Counts of the reference radix-4 loops (nttcore.py:200-257, 267-323)."""
    c = _counts()
    if not inverse:
        m, k = 1, n // 2
        while m < n:
            c[C_TWIDDLE] += 3 * m
            c[C_MODMUL] += m * 4 * (k // 2)
            c[C_ADDSUB] += m * 8 * (k // 2)
            m, k = m << 2, k >> 2
    else:
        m, k = n // 2, 1
        while m >= 2:
            g = m // 2
            c[C_TWIDDLE] += 3 * g
            c[C_MODMUL] += g * 4 * k
            c[C_ADDSUB] += g * 8 * k
            c[C_HALF] += g * 8 * k
            m, k = m >> 2, k << 2
    return c


def ntt_radix4(a: Polynomial, plan: NttPlan, ctr: OpCounter | None = None) -> Polynomial:
    """Forward NTT, two stages per pass; requires even log2(n)."""
    if plan.log_n % 2:
        raise ValueError(f"radix-4 needs even log2(n), got n={plan.n}")
    _check(a, plan, NORMAL)
    backend.kernels().ntt_ct(a.coeffs, plan.tw_fwd, *plan.red_args, False, None)
    _finish(ctr, _radix4_counts(plan.n, False))
    a.ordering = BIT_REVERSED
    return a


def intt_radix4(a: Polynomial, plan: NttPlan, ctr: OpCounter | None = None) -> Polynomial:
    """Scaled inverse paired with ntt_radix4; requires even log2(n)."""
    if plan.log_n % 2:
        raise ValueError(f"radix-4 needs even log2(n), got n={plan.n}")
    _check(a, plan, BIT_REVERSED)
    q, mode, mu, s_in, s_out = plan.red_args
    backend.kernels().intt_gs(a.coeffs, plan.tw_inv, q, plan.mod.half_q_ceil, mode, mu, s_in,
                              s_out, True, False, None)
    _finish(ctr, _radix4_counts(plan.n, True))
    a.ordering = NORMAL
    return a


# ---------------------------------------------------------------------------
# four-step 2D shape (reference nttcore.py:332-497).  Its output is the
# natural-order negacyclic spectrum in the "vendor order" (entry j2 + n2*j1
# at position j2*n1 + j1), i.e. a fixed permutation of the merged-CT output
# (ntt_2d_permutation).  The GPU computes the merged transform with its
# stage-grouped 2D schedule and applies the permutation with one gather
# launch; the inverse gathers back and runs the scaled merged inverse.

def _grid_split(plan: NttPlan) -> tuple[int, int]:
    if plan.log_n % 2 == 0:
        return 1 << (plan.log_n // 2), 1 << (plan.log_n // 2)
    return 1 << ((plan.log_n + 1) // 2), 1 << ((plan.log_n - 1) // 2)


def ntt_2d_permutation(plan: NttPlan) -> np.ndarray:
    """perm such that ntt_2d(a).coeffs[v] == ntt_ct(a).coeffs[perm[v]]."""
    cached = plan._cache.get("2d_perm")
    if cached is None:
        n1, n2 = _grid_split(plan)
        v = np.arange(plan.n, dtype=np.int64)
        j2, j1 = np.divmod(v, n1)
        idx = j2 + n2 * j1
        rev = np.zeros(plan.n, dtype=np.int64)
        for bit in range(plan.log_n):  # bit reversal of log_n-bit indices
            rev |= ((idx >> bit) & 1) << (plan.log_n - 1 - bit)
        cached = rev
        plan._cache["2d_perm"] = cached
    return cached.copy()


def _perm_device(plan: NttPlan, inverse: bool) -> torch.Tensor:
    key = "2d_perm_inv_dev" if inverse else "2d_perm_dev"
    t = plan._cache.get(key)
    if t is None:
        perm = ntt_2d_permutation(plan)
        if inverse:
            inv = np.empty_like(perm)
            inv[perm] = np.arange(plan.n, dtype=np.int64)
            perm = inv
        t = torch.from_numpy(perm).to(_device.device())
        plan._cache[key] = t
    return t


def _counts_2d_one(plan: NttPlan) -> np.ndarray:
    """Counts of one ntt_2d / ntt_2d_inv (reference nttcore.py:405-486): n
    pre/post products, n twiddle corrections, (n/2) log2 n butterflies."""
    n, log_n = plan.n, plan.log_n
    c = _counts()
    c[C_MODMUL] = 2 * n + (n // 2) * log_n
    c[C_TWIDDLE] = 2 * n + (n // 2) * log_n
    c[C_ADDSUB] = n * log_n
    return c


def ntt_2d(a: Polynomial, plan: NttPlan, ctr: OpCounter | None = None) -> Polynomial:
    """Four-step forward transform: normal order in, vendor order out."""
    _check(a, plan, NORMAL)
    k = backend.kernels()
    work = a.coeffs.clone()
    k.ntt_ct(work, plan.tw_fwd, *plan.red_args, False, None)
    a.coeffs = k.gather(work, _perm_device(plan, False))
    a.ordering = VENDOR_2D
    _finish(ctr, _counts_2d_one(plan))
    return a


def ntt_2d_inv(a: Polynomial, plan: NttPlan, ctr: OpCounter | None = None) -> Polynomial:
    """Inverse of ntt_2d, consuming its vendor order (scaled: returns the input)."""
    if len(a.coeffs) != plan.n:
        raise ValueError(f"length {len(a.coeffs)} does not match plan n={plan.n}")
    if a.ordering != VENDOR_2D:
        raise ValueError(f"expected vendor_2d-order input, got {a.ordering}")
    k = backend.kernels()
    work = k.gather(a.coeffs, _perm_device(plan, True))
    q, mode, mu, s_in, s_out = plan.red_args
    k.intt_gs(work, plan.tw_inv, q, plan.mod.half_q_ceil, mode, mu, s_in, s_out, True, False,
              None)
    a.coeffs = work
    a.ordering = NORMAL
    _finish(ctr, _counts_2d_one(plan))
    return a


def _stack(rows: list[Polynomial], n: int) -> torch.Tensor:
    for r in rows:
        if len(r) != n:
            raise ValueError("ragged batch: all rows must have length n")
    return torch.stack([r.coeffs for r in rows]) if rows else None


def batch_ntt(rows: list[Polynomial], plan: NttPlan, workers: int = 1,
              ctr: OpCounter | None = None) -> list[Polynomial]:
    """ntt_ct on every row with one [B, n] launch; deterministic for any workers."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    block = _stack(rows, plan.n)
    if block is None:
        return rows
    for r in rows:
        _check(r, plan, NORMAL)
    counts = _counts()
    backend.kernels().ntt_ct(block, plan.tw_fwd, *plan.red_args, False, counts)
    for i, r in enumerate(rows):
        r.coeffs = block[i]
        r.ordering = BIT_REVERSED
    _finish(ctr, counts)
    return rows


def batch_intt(rows: list[Polynomial], plan: NttPlan, scaled: bool = True,
               ctr: OpCounter | None = None) -> list[Polynomial]:
    """Batched inverse (extension): one launch over [B, n]."""
    block = _stack(rows, plan.n)
    if block is None:
        return rows
    for r in rows:
        _check(r, plan, BIT_REVERSED)
    q, mode, mu, s_in, s_out = plan.red_args
    counts = _counts()
    backend.kernels().intt_gs(block, plan.tw_inv, q, plan.mod.half_q_ceil, mode, mu, s_in,
                              s_out, scaled, False, counts)
    for i, r in enumerate(rows):
        r.coeffs = block[i]
        r.ordering = NORMAL
    _finish(ctr, counts)
    return rows
