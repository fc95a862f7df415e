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
