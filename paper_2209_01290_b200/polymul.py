"""Negacyclic polynomial products on the GPU (reference pkg/src/nttmul/polymul.py).

``polymul_fused`` is the north-star unit of work: truncated forward NTTs of
a and b, the Karatsuba-fused middle (paper Alg. 8) and the truncated scaled
inverse.  Where the reference makes four kernel calls per product
(polymul.py:163-169), here the whole product is ONE call of the C ABI
``nttmul_polymul_fused_rns`` (column pass, fused row kernel, inverse column
pass for n > 4096; a single row kernel otherwise).

Return types follow the inputs: CUDA-tensor (or Polynomial) operands give a
CUDA tensor; lists / numpy arrays give a numpy array (host-buffer path:
staged to HBM and back, as the reference returns ndarrays).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib, backend
from .modarith import Modulus, mod_add, mod_sub, mulmod
from .nttcore import (
    NORMAL,
    OpCounter,
    Polynomial,
    _counts,
    _finish,
)
from .params import NttPlan

TRANSFORMS = ("radix2", "radix4", "2d")


@dataclass(frozen=True)
class FusedPlan:
    """A plan plus the halved twiddle tables the fused path reads.

    Fusion never touches the upper half of either table, so only n/2 forward
    and n/2 inverse words (views of the plan's device tables) are kept.
    """

    base: NttPlan
    tw_fwd_half: torch.Tensor
    tw_inv_half: torch.Tensor
    fwd_pairs_half: torch.Tensor
    inv_pairs_half: torch.Tensor

    @classmethod
    def from_plan(cls, plan: NttPlan) -> "FusedPlan":
        key = ("fused", _device.device().index)  # views of this device's tables
        cached = plan._cache.get(key)
        if cached is None:
            h = plan.n // 2
            cached = cls(base=plan, tw_fwd_half=plan.tw_fwd[:h], tw_inv_half=plan.tw_inv[:h],
                         fwd_pairs_half=plan.fwd_pairs[:h], inv_pairs_half=plan.inv_pairs[:h])
            plan._cache[key] = cached
        return cached

    @property
    def mode(self) -> int:
        """C-ABI reduction mode with the lazy-bound flags of this prime."""
        m = self.base._cache.get("fused_mode")
        if m is None:
            m = self.base._cache["fused_mode"] = mode_flags(self.base.red_args[1], [self.base.q])
        return m

    def workspace(self) -> torch.Tensor | None:
        """Scratch of one limb-product for the column passes (n > 4096),
        kept per device and stream: calls on one stream are ordered, so they
        can share it (a fresh allocation per call costs host time)."""
        if self.base.log_n <= 12:
            return None
        key = ("fused_ws", _device.index(), _device.stream_ptr())
        ws = self.base._cache.get(key)
        if ws is None:
            ws = self.base._cache[key] = torch.empty(self.base.n, dtype=_device.U64,
                                                     device=_device.device())
        return ws


def _coeffs(a, n: int):
    """(device tensor, came_from_device) of a normal-order operand."""
    if isinstance(a, Polynomial):
        if a.ordering != NORMAL:
            raise ValueError(f"expected normal-order input, got {a.ordering}")
        t, dev = a.coeffs, True
    else:
        dev = _device.is_device_tensor(a)
        t = _device.to_device(a)
    if t.dim() != 1 or t.numel() != n:
        raise ValueError(f"length {t.numel()} does not match n={n}")
    return t, dev


def _result(t: torch.Tensor, on_device: bool):
    return t if on_device else t.cpu().numpy()


def negacyclic_naive(a, b, q: int, ctr: OpCounter | None = None):
    """Schoolbook product mod x^n + 1; the independent O(n^2) oracle,
    reduced by division only (reference polymul.py:70-82).  One GPU thread
    per output coefficient; [batch, n] device tensors run as one launch."""
    dev = _device.is_device_tensor(a) or _device.is_device_tensor(b)
    ta, tb = _device.to_device(a), _device.to_device(b)
    if ta.shape[-1] != tb.shape[-1] or ta.shape != tb.shape:
        raise ValueError(f"length mismatch: {ta.shape[-1]} vs {tb.shape[-1]}")
    out = torch.empty_like(ta)
    counts = _counts()
    backend.kernels().negacyclic_naive(ta, tb, out, int(q), counts)
    _finish(ctr, counts)
    return _result(out, dev)


def hadamard(a, b, mod_or_plan, ctr: OpCounter | None = None):
    """Entry-wise modular product of two equal-length vectors."""
    if isinstance(mod_or_plan, NttPlan):
        q, mode, mu, s_in, s_out = mod_or_plan.red_args
    else:
        mod: Modulus = mod_or_plan
        q = mod.q
        mode, mu, s_in, s_out = mod.reduction_params("proposed")
    dev = _device.is_device_tensor(a) or _device.is_device_tensor(b)
    ta, tb = _device.to_device(a), _device.to_device(b)
    if ta.numel() != tb.numel():
        raise ValueError(f"length mismatch: {ta.numel()} vs {tb.numel()}")
    out = torch.empty_like(ta)
    counts = _counts()
    backend.kernels().hadamard(ta, tb, out, q, mode, mu, s_in, s_out, counts)
    _finish(ctr, counts)
    return _result(out, dev)


def _counts_2d(plan: NttPlan, ctr: OpCounter) -> None:
    """Reference bookkeeping of polymul_ntt(transform="2d"): ntt_2d twice,
    hadamard, ntt_2d_inv (nttcore.py:405-486).  Each 2D transform does n
    pre/post products, n twiddle corrections and (n/2) log2 n butterflies."""
    n, log_n = plan.n, plan.log_n
    per = 2 * n + (n // 2) * log_n
    ctr.modmul += 3 * per + n
    ctr.twiddle_loads += 3 * per
    ctr.modadd_sub += 3 * n * log_n


def polymul_ntt(a, b, plan: NttPlan, ctr: OpCounter | None = None,
                transform: str = "radix2"):
    """Eq. (2): forward transforms, pointwise product, scaled inverse.

    All three reference transform shapes give bit-identical products (the
    reference's own test_alternate_transforms); on the GPU each runs the
    radix-2 merged kernels, whose schedule already groups stages by radix.
    Counts follow the requested shape's reference bookkeeping.
    """
    if transform not in TRANSFORMS:
        raise ValueError(f"unknown transform {transform!r}")
    ta, dev_a = _coeffs(a, plan.n)
    tb, dev_b = _coeffs(b, plan.n)
    k = backend.kernels()
    q, mode, mu, s_in, s_out = plan.red_args
    block = torch.stack([ta, tb])  # copies: inputs are preserved
    counts = _counts()
    k.ntt_ct(block, plan.tw_fwd, q, mode, mu, s_in, s_out, False, counts)
    spec = torch.empty_like(ta)
    k.hadamard(block[0], block[1], spec, q, mode, mu, s_in, s_out, counts)
    k.intt_gs(spec, plan.tw_inv, q, plan.mod.half_q_ceil, mode, mu, s_in, s_out, True, False,
              counts)
    if ctr is not None:
        if transform == "2d":
            _counts_2d(plan, ctr)
        else:  # radix-4 bookkeeping equals radix-2 (reference test_nttcore.py:129-138)
            ctr.add_array(counts)
    return _result(spec, dev_a or dev_b)


def fused_butterfly(a0: int, a1: int, b0: int, b1: int, alpha_sq: int, mod: Modulus,
                    ctr: OpCounter | None = None, variant: str = "proposed"):
    """Scalar Alg. 7 component: (a0 b0 + alpha^2 a1 b1, a0 b1 + a1 b0) mod q with
    4 products and 5 sums (host reference semantics, polymul.py:126-144)."""
    u = mulmod(a0, b0, mod, variant)
    v = mulmod(a1, b1, mod, variant)
    w = mulmod(mod_add(a0, a1, mod), mod_add(b0, b1, mod), mod, variant)
    z = mulmod(alpha_sq, v, mod, variant)
    if ctr is not None:
        ctr.modmul += 4
        ctr.modadd_sub += 5
    return mod_add(u, z, mod), mod_sub(mod_sub(w, u, mod), v, mod)


def _fused_counts(n: int, batch: int = 1) -> np.ndarray:
    """Reference counts of one polymul_fused (probe-verified closed form)."""
    lg = n.bit_length() - 1
    c = np.zeros(5, dtype=np.uint64)
    c[0] = batch * ((3 * n // 2) * (lg - 1) + 2 * n)
    c[1] = batch * (3 * n * (lg - 1) + 5 * n // 2)
    c[2] = batch * (n * (lg - 1))
    c[3] = batch * (2 * n - 3)
    c[4] = batch * (n // 4)
    return c


MODE_NARROW = 0x100    # NTTMUL_MODE_NARROW: every modulus < 2^61 ([0, 8q) lazy bound)
MODE_NARROW60 = 0x200  # NTTMUL_MODE_NARROW60: every modulus < 2^60 ([0, 16q) forward)


MODE_WIDE35 = 0x400    # NTTMUL_MODE_WIDE35: every modulus >= 2^34 (multiply-based reductions)


def mode_flags(mode: int, primes) -> int:
    """Reduction mode plus the lazy-bound flags the moduli allow."""
    top = max(primes)
    if top < (1 << 60):
        wide = MODE_WIDE35 if min(primes).bit_length() >= 35 else 0
        return mode | MODE_NARROW | MODE_NARROW60 | wide
    return mode | (MODE_NARROW if top < (1 << 61) else 0)


def run_fused(out: torch.Tensor, a: torch.Tensor, b: torch.Tensor, fwd_pairs, inv_pairs,
              limbs_dev: torch.Tensor, log_n: int, num_limbs: int, batch: int, mode: int,
              workspace: torch.Tensor | None = None) -> None:
    """Launch the fused RNS polymul over [batch, num_limbs, n] device tensors."""
    if log_n > 12 and workspace is None:  # column passes need scratch (n > row length)
        workspace = torch.empty_like(a)
    _lib.call("nttmul_polymul_fused_rns", out.data_ptr(), a.data_ptr(), b.data_ptr(),
              limbs_dev.data_ptr(), fwd_pairs.data_ptr(), inv_pairs.data_ptr(), log_n,
              num_limbs, batch, mode, _device.ptr(workspace), _device.stream_ptr())


def _fused_fast(a: torch.Tensor, b: torch.Tensor, fused: FusedPlan):
    """One limb-product of contiguous CUDA uint64 [n] operands with the
    plan's cached device pointers (a single product's Python overhead is
    otherwise comparable to its device time); None -> the general path."""
    base = fused.base
    n = base.n
    if (a.dtype is not _device.U64 or b.dtype is not _device.U64 or not a.is_cuda
            or not b.is_cuda or a.shape != (n,) or b.shape != (n,)
            or not a.is_contiguous() or not b.is_contiguous() or a.device != b.device):
        return None
    key = ("fused_fast", a.device.index)
    c = base._cache.get(key)
    if c is None:
        c = base._cache[key] = (fused.fwd_pairs_half.data_ptr(), fused.inv_pairs_half.data_ptr(),
                                base.limb_device().data_ptr(), fused.mode, base.log_n)
    out = torch.empty_like(a)
    ws = fused.workspace()
    st = _lib.load().nttmul_polymul_fused_rns(
        out.data_ptr(), a.data_ptr(), b.data_ptr(), c[2], c[0], c[1], c[4], 1, 1, c[3],
        0 if ws is None else ws.data_ptr(), _device.stream_ptr())
    if st:
        _lib.check(st, "nttmul_polymul_fused_rns")
    return out


def polymul_fused(a, b, plan: NttPlan | FusedPlan, ctr: OpCounter | None = None):
    """Negacyclic product through the fused pipeline (one GPU call).

    For n = 2 there is no stage to truncate and the unfused pipeline is used
    (reference polymul.py:156-157).
    """
    fused = plan if isinstance(plan, FusedPlan) else FusedPlan.from_plan(plan)
    base = fused.base
    if base.n < 4:
        return polymul_ntt(a, b, base, ctr)
    if ctr is None and type(a) is torch.Tensor and type(b) is torch.Tensor:
        out = _fused_fast(a, b, fused)
        if out is not None:
            return out
    ta, dev_a = _coeffs(a, base.n)
    tb, dev_b = _coeffs(b, base.n)
    out = torch.empty_like(ta)
    run_fused(out, ta, tb, fused.fwd_pairs_half, fused.inv_pairs_half, base.limb_device(),
              base.log_n, 1, 1, fused.mode, fused.workspace())
    _finish(ctr, _fused_counts(base.n))
    return _result(out, dev_a or dev_b)


def polymul_batch(pairs, plan: NttPlan | FusedPlan, workers: int = 1,
                  ctr: OpCounter | None = None):
    """Independent fused products as ONE [B, n] launch (any ``workers``)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    fused = plan if isinstance(plan, FusedPlan) else FusedPlan.from_plan(plan)
    base = fused.base
    n = base.n
    for a, b in pairs:
        if len(a) != n or len(b) != n:
            raise ValueError("ragged batch: all operands must have length n")
    if not pairs:
        return []
    if n < 4:
        return [polymul_fused(a, b, fused, ctr) for a, b in pairs]
    cols_a, cols_b, dev = [], [], False
    for a, b in pairs:
        ta, da = _coeffs(a, n)
        tb, db = _coeffs(b, n)
        cols_a.append(ta)
        cols_b.append(tb)
        dev = dev or da or db
    A, Bm = torch.stack(cols_a), torch.stack(cols_b)
    out = torch.empty_like(A)
    run_fused(out, A, Bm, fused.fwd_pairs_half, fused.inv_pairs_half, base.limb_device(),
              base.log_n, 1, len(pairs), mode_flags(base.red_args[1], [base.q]))
    _finish(ctr, _fused_counts(n, len(pairs)))
    return [_result(out[i], dev) for i in range(len(pairs))]
