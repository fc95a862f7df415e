"""The kernel surface - drop-in for the reference's ``nttmul._kernels``.

Same function names, argument order and in-place / accumulate semantics as
/root/reference/pkg/src/nttmul/_kernels.pyx (what ``backend.kernels()``
returns there), executed by the sm_100a library through the C ABI:

  ntt_ct(a, tw, q, mode, mu, s_in, s_out, truncate, counts)        pyx:52-85
  intt_gs(a, tw, q, half_q, mode, mu, s_in, s_out, scaled,
          skip_first, counts)                                      pyx:88-129
  fused_middle(ah, bh, ch, tw, q, mode, mu, s_in, s_out, counts)   pyx:132-177
  hadamard(a, b, out, q, mode, mu, s_in, s_out, counts)            pyx:180-188
  scale(a, factor, q, mode, mu, s_in, s_out, counts)               pyx:191-199
  mulmod_loop(a, b, q, mode, mu, s_in, s_out, passes) -> int       pyx:359-371
  negacyclic_naive(a, b, out, q, counts)                           pyx:200-223
  sweep_exhaustive(q_lo, q_hi, tallies) -> (mism, first)           pyx:264-306
  sweep_random(bits, nsamples, seed, tallies) -> (mism, first)     pyx:309-356

Operands may be CUDA uint64 tensors (1-D ``[n]`` as in the reference, or
``[batch, n]`` to transform a whole batch in one launch) or numpy uint64
arrays (staged to the device and written back in place - the host-buffer
path).  ``counts`` (uint64[5]: modmul, addsub, half, twiddle loads,
negations) is accumulated with the reference's closed forms, which are
data-independent.  Launches go to torch's current stream.

The verification kernels (schoolbook oracle, reduction sweeps) run on the
GPU too (csrc/verify_kernels.cuh) with the reference's exact arithmetic;
the sweeps' ``tallies`` (uint64[3][4]) are accumulated like the reference.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np
import torch

from . import _device, _lib

NATIVE = True

C_MODMUL, C_ADDSUB, C_HALF, C_TWIDDLE, C_NEG = range(5)
RED_BUILTIN, RED_TWO_SUB, RED_ONE_SUB = 0, 1, 2

# ---------------------------------------------------------------------------
# twiddle pair tables: {w, floor(w 2^64 / q)} per entry, cached per table
#
# Entries are keyed by the identity of the caller's table (a CUDA tensor or a
# numpy array) and evicted when that table is garbage-collected
# (weakref.finalize), so the cache never keeps a plan's tables alive.  A
# device table is re-paired when its torch version counter moved (in-place
# edit); a host table when its contents differ from the copy taken when it
# was paired (the reference passes plain ndarrays on every call, so a numpy
# caller pays one host compare instead of an upload + pairing launch).  At
# most _PAIRS_MAX foreign tables are cached (oldest dropped first).

_PAIRS: dict = {}
_PAIRS_MAX = 64
_PAIRS_LOCK = threading.RLock()  # re-entrant: a finalizer may run inside a locked section


def _evict(key) -> None:
    with _PAIRS_LOCK:
        _PAIRS.pop(key, None)


def _remember(tw, q: int, entry) -> None:
    key = (id(tw), q, _device.index())
    with _PAIRS_LOCK:
        fresh = key not in _PAIRS
        if fresh:
            while len(_PAIRS) >= _PAIRS_MAX:
                _PAIRS.pop(next(iter(_PAIRS)))
        _PAIRS[key] = entry
    if fresh:
        weakref.finalize(tw, _evict, key)


def register_pairs(tw: torch.Tensor, pairs: torch.Tensor, q: int, w1: int) -> None:
    """Record the pair table (and tw[1]) that belongs to device table ``tw``
    (the caller - a plan - owns both; the cache holds no strong reference).
    The table is also attached to ``tw`` itself for the transforms' fast
    path (``tw`` keeps its own pair table alive, nothing else)."""
    _remember(tw, q, (tw._version, weakref.ref(pairs), w1, None))
    tw._nttb_pairs = (int(q), tw._version, pairs.data_ptr(), int(w1), pairs.shape[0], pairs)


# ---------------------------------------------------------------------------
# fast path of the transforms: a contiguous CUDA uint64 [n] / [batch, n]
# operand and a plan's device twiddle table with its attached pair table.
# Skips the general operand / cache machinery (a single transform's Python
# overhead is otherwise larger than its device time); any other argument
# takes the general path below, which also produces the errors.

_FNS: dict = {}


def _fn(name: str):
    f = _FNS.get(name)
    if f is None:
        f = _FNS[name] = getattr(_lib.load(), name)
    return f


def _fast(a, tw, q):
    """(data ptr, batch, log_n, pairs ptr, pair entries, w1) or None."""
    if type(a) is not torch.Tensor or type(tw) is not torch.Tensor:
        return None
    e = tw.__dict__.get("_nttb_pairs")
    if e is None or e[0] != q or e[1] != tw._version:
        return None
    if a.dtype is not _device.U64 or not a.is_cuda or not a.is_contiguous():
        return None
    sh = a.shape
    if len(sh) == 1:
        batch, n = 1, sh[0]
    elif len(sh) == 2:
        batch, n = sh
    else:
        return None
    if n < 2 or n & (n - 1):
        return None
    return a.data_ptr(), batch, n.bit_length() - 1, e[2], e[4], e[3]


def _lookup(tw, q: int):
    hit = _PAIRS.get((id(tw), q, _device.index()))
    if hit is None:
        return None
    version, pref, w1, host_copy = hit
    pairs = pref() if isinstance(pref, weakref.ref) else pref
    if pairs is None:
        return None
    if isinstance(tw, torch.Tensor):
        return (pairs, w1) if version == tw._version else None
    return (pairs, w1) if host_copy.shape == tw.shape and np.array_equal(host_copy, tw) else None


def _pairs_for(tw, q: int):
    """(pairs tensor, tw[1]) for a twiddle table given as tensor or ndarray."""
    cacheable = (isinstance(tw, torch.Tensor) and tw.is_cuda) or isinstance(tw, np.ndarray)
    if cacheable:
        hit = _lookup(tw, q)
        if hit is not None:
            return hit
    t = _device.to_device(tw)
    pairs = torch.empty((t.numel(), 2), dtype=_device.U64, device=t.device)
    _lib.call("nttmul_shoup_pairs", pairs.data_ptr(), t.data_ptr(), q, t.numel(),
              _device.stream_ptr())
    w1 = int(t[1].item()) if t.numel() > 1 else 1
    if isinstance(tw, torch.Tensor) and tw.is_cuda:
        _remember(tw, q, (tw._version, pairs, w1, None))
        if pairs.device == tw.device:  # (the transforms' fast path)
            tw._nttb_pairs = (q, tw._version, pairs.data_ptr(), w1, pairs.shape[0], pairs)
    elif isinstance(tw, np.ndarray):
        _remember(tw, q, (None, pairs, w1, np.array(tw, dtype=np.uint64, copy=True)))
    return pairs, w1


# ---------------------------------------------------------------------------
# operands

class _Operand:
    """A device view of an argument; numpy arguments are written back."""

    __slots__ = ("host", "dev")

    def __init__(self, x, name: str, writable: bool = True):
        if isinstance(x, torch.Tensor):
            if x.dtype != _device.U64:
                raise ValueError(f"{name}: expected uint64, got {x.dtype}")
            if not x.is_cuda:
                raise ValueError(f"{name}: CPU tensors are not accepted; use a CUDA tensor "
                                 "or a numpy array")
            if not x.is_contiguous():
                raise ValueError(f"{name}: tensor must be contiguous")
            self.host, self.dev = None, x
        elif isinstance(x, np.ndarray):
            if x.dtype != np.uint64:
                raise ValueError(f"{name}: Buffer dtype mismatch, expected uint64, got {x.dtype}")
            if not x.flags.c_contiguous:
                raise ValueError(f"{name}: ndarray is not C-contiguous")
            if writable and not x.flags.writeable:
                raise ValueError(f"{name}: buffer source array is read-only")
            self.host = x
            self.dev = torch.from_numpy(x).to(_device.device())
        else:
            raise TypeError(f"{name}: a bytes-like uint64 buffer or CUDA tensor is required, "
                            f"not {type(x).__name__}")

    def writeback(self) -> None:
        if self.host is not None:
            self.host[...] = self.dev.cpu().numpy()


def _shape(op: _Operand) -> tuple[int, int]:
    """(batch, n) of a [n] or [batch, n] operand."""
    t = op.dev
    if t.dim() == 1:
        return 1, t.shape[0]
    if t.dim() == 2:
        return t.shape[0], t.shape[1]
    raise ValueError("operands are [n] or [batch, n]")


def _log2(n: int, what: str = "length") -> int:
    if n < 1 or n & (n - 1):
        raise ValueError(f"{what} {n} is not a power of two")
    return n.bit_length() - 1


def _add_counts(counts, vals) -> None:
    if counts is None:
        return
    for i, v in enumerate(vals):
        if v:
            counts[i] += np.uint64(v)


# closed-form operation counts of the reference kernels (data-independent)

def _fwd_counts(n: int, truncate: bool):
    limit = n // 2 if truncate else n
    m, stages, groups = 1, 0, 0
    while m < limit:
        stages += 1
        groups += m
        m <<= 1
    return (n // 2) * stages, stages, groups


def _inv_counts(n: int, skip: bool):
    m = n // 4 if skip else n // 2
    stages, groups = 0, 0
    while m >= 1:
        stages += 1
        groups += m
        m >>= 1
    return (n // 2) * stages, stages, groups


# ---------------------------------------------------------------------------
# the surface

def ntt_ct(a, tw, q, mode, mu, s_in, s_out, truncate, counts=None):
    """Merged CT forward NTT in place (normal -> bit-reversed order)."""
    f = _fast(a, tw, q) if counts is None else None
    if f is not None and f[4] >= max((1 << f[2]) >> (1 if truncate else 0), 2):
        st = _fn("nttmul_ntt_ct")(f[0], f[3], int(q), int(mode), int(mu), int(s_in), int(s_out),
                                  1 if truncate else 0, f[2], f[1], _device.stream_ptr())
        if st:
            _lib.check(st, "nttmul_ntt_ct")
        return
    op = _Operand(a, "a")
    batch, n = _shape(op)
    log_n = _log2(n)
    need = n // 2 if truncate else n
    pairs, _ = _pairs_for(tw, int(q))
    if pairs.shape[0] < max(need, 2):
        raise ValueError(f"twiddle table has {pairs.shape[0]} entries, transform needs {need}")
    _lib.call("nttmul_ntt_ct", op.dev.data_ptr(), pairs.data_ptr(), int(q), int(mode), int(mu),
              int(s_in), int(s_out), int(bool(truncate)), log_n, batch, _device.stream_ptr())
    op.writeback()
    if counts is not None:
        mul, _, groups = _fwd_counts(n, bool(truncate))
        _add_counts(counts, (batch * mul, 2 * batch * mul, 0, batch * groups, 0))


def intt_gs(a, tw, q, half_q, mode, mu, s_in, s_out, scaled, skip_first, counts=None):
    """Merged GS inverse NTT in place (bit-reversed -> normal order)."""
    f = _fast(a, tw, q) if counts is None else None
    if f is not None and f[4] >= max((1 << f[2]) >> (1 if skip_first else 0), 2):
        st = _fn("nttmul_intt_gs")(f[0], f[3], int(q), int(half_q), int(mode), int(mu),
                                   int(s_in), int(s_out), 1 if scaled else 0,
                                   1 if skip_first else 0, f[2], f[1], f[5],
                                   _device.stream_ptr())
        if st:
            _lib.check(st, "nttmul_intt_gs")
        return
    op = _Operand(a, "a")
    batch, n = _shape(op)
    log_n = _log2(n)
    need = n // 2 if skip_first else n
    pairs, w1 = _pairs_for(tw, int(q))
    if pairs.shape[0] < max(need, 2):
        raise ValueError(f"twiddle table has {pairs.shape[0]} entries, transform needs {need}")
    _lib.call("nttmul_intt_gs", op.dev.data_ptr(), pairs.data_ptr(), int(q), int(half_q),
              int(mode), int(mu), int(s_in), int(s_out), int(bool(scaled)),
              int(bool(skip_first)), log_n, batch, w1, _device.stream_ptr())
    op.writeback()
    if counts is not None:
        mul, _, groups = _inv_counts(n, bool(skip_first))
        _add_counts(counts, (batch * mul, 2 * batch * mul, 2 * batch * mul if scaled else 0,
                             batch * groups, 0))


def fused_middle(ah, bh, ch, tw, q, mode, mu, s_in, s_out, counts=None):
    """Karatsuba-fused last-CT / pointwise / first-GS stage (Alg. 8)."""
    oa, ob, oc = _Operand(ah, "ah", False), _Operand(bh, "bh", False), _Operand(ch, "ch")
    batch, n = _shape(oa)
    if _shape(ob) != (batch, n) or _shape(oc) != (batch, n):
        raise ValueError("ah, bh, ch must share one shape")
    log_n = _log2(n)
    if n < 4:
        raise ValueError("fused middle needs n >= 4")
    pairs, _ = _pairs_for(tw, int(q))
    _lib.call("nttmul_fused_middle", oa.dev.data_ptr(), ob.dev.data_ptr(), oc.dev.data_ptr(),
              pairs.data_ptr(), int(q), int(mode), int(mu), int(s_in), int(s_out), log_n,
              batch, _device.stream_ptr())
    oc.writeback()
    half = n // 2
    _add_counts(counts, (4 * half * batch, 5 * half * batch, 0, half * batch,
                         (half // 2) * batch))


def hadamard(a, b, out, q, mode, mu, s_in, s_out, counts=None):
    """out = a * b mod q entry-wise."""
    oa, ob, oo = _Operand(a, "a", False), _Operand(b, "b", False), _Operand(out, "out")
    n = oa.dev.numel()
    if ob.dev.numel() != n or oo.dev.numel() != n:
        raise ValueError("a, b, out must have equal length")
    _lib.call("nttmul_hadamard", oa.dev.data_ptr(), ob.dev.data_ptr(), oo.dev.data_ptr(), n,
              int(q), int(mode), int(mu), int(s_in), int(s_out), _device.stream_ptr())
    oo.writeback()
    _add_counts(counts, (n, 0, 0, 0, 0))


def scale(a, factor, q, mode, mu, s_in, s_out, counts=None):
    """a = a * factor mod q in place."""
    op = _Operand(a, "a")
    n = op.dev.numel()
    _lib.call("nttmul_scale", op.dev.data_ptr(), int(factor), n, int(q), int(mode), int(mu),
              int(s_in), int(s_out), _device.stream_ptr())
    op.writeback()
    _add_counts(counts, (n, 0, 0, 0, 0))


def mulmod_loop(a, b, q, mode, mu, s_in, s_out, passes) -> int:
    """XOR over ``passes`` passes of a[i]*b[i] mod q (the reference bench loop)."""
    oa, ob = _Operand(a, "a", False), _Operand(b, "b", False)
    n = oa.dev.numel()
    if ob.dev.numel() != n:
        raise ValueError("a and b must have equal length")
    sink = torch.zeros(1, dtype=_device.U64, device=oa.dev.device)
    _lib.call("nttmul_mulmod_loop", oa.dev.data_ptr(), ob.dev.data_ptr(), n, int(q), int(mode),
              int(mu), int(s_in), int(s_out), int(passes), sink.data_ptr(),
              _device.stream_ptr())
    return int(sink.item())


def mulmod_tensor(a, b, mod, variant: str = "proposed") -> torch.Tensor:
    """Element-wise a*b mod q of two CUDA tensors (modarith.mulmod device path)."""
    da, db = _device.to_device(a), _device.to_device(b)
    if da.shape != db.shape:
        raise ValueError(f"shape mismatch: {tuple(da.shape)} vs {tuple(db.shape)}")
    out = torch.empty_like(da)
    mode, mu, s_in, s_out = mod.reduction_params(variant)
    _lib.call("nttmul_hadamard", da.data_ptr(), db.data_ptr(), out.data_ptr(), da.numel(),
              mod.q, mode, mu, s_in, s_out, _device.stream_ptr())
    return out


def negacyclic_naive(a, b, out, q, counts=None):
    """Schoolbook product mod x^n + 1 (division-based reduction only)."""
    oa, ob, oo = _Operand(a, "a", False), _Operand(b, "b", False), _Operand(out, "out")
    batch, n = _shape(oa)
    if _shape(ob) != (batch, n) or _shape(oo) != (batch, n):
        raise ValueError("a, b, out must share one shape")
    _lib.call("nttmul_negacyclic_naive", oo.dev.data_ptr(), oa.dev.data_ptr(),
              ob.dev.data_ptr(), int(q), n, batch, _device.stream_ptr())
    oo.writeback()
    _add_counts(counts, (batch * n * n, batch * n * n, 0, 0, 0))


def _sweep_finish(tallies, t_dev, r_dev):
    t = t_dev.cpu().numpy().reshape(3, 4)
    res = r_dev.cpu().numpy()
    if isinstance(tallies, torch.Tensor):
        tallies += torch.from_numpy(t.astype(np.uint64)).to(tallies.device)
    else:
        tallies[...] = np.asarray(tallies, dtype=np.uint64) + t.astype(np.uint64)
    return int(res[0]), int(res[1])


_MASK64 = (1 << 64) - 1


def _splitmix_at(seed: int, draws: int) -> int:
    z = (seed + draws * 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def sweep_exhaustive(q_lo, q_hi, tallies):
    """All odd q in [q_lo, q_hi], all x < q^2, every Barrett variant against
    division; tallies uint64[3][4] += counts of 0/1/2/3+ subtractions.
    Returns (mismatches, (q, x, variant) of the first mismatch or None)."""
    dev = _device.device()
    t_dev = torch.empty(12, dtype=_device.U64, device=dev)
    r_dev = torch.empty(2, dtype=_device.U64, device=dev)
    _lib.call("nttmul_sweep_exhaustive", int(q_lo), int(q_hi), t_dev.data_ptr(),
              r_dev.data_ptr(), _device.stream_ptr())
    mism, key = _sweep_finish(tallies, t_dev, r_dev)
    if not mism:
        return 0, None
    qi, x, vi = key >> 34, (key >> 2) & ((1 << 32) - 1), key & 3
    return mism, ((int(q_lo) | 1) + 2 * qi, x, vi)


def sweep_random(bits, nsamples, seed, tallies):
    """Random (a, b, q) triples (splitmix64 stream of the reference) with q an
    odd ``bits``-bit modulus; same return convention as sweep_exhaustive
    (first = (q, a*b, variant))."""
    dev = _device.device()
    t_dev = torch.empty(12, dtype=_device.U64, device=dev)
    r_dev = torch.empty(2, dtype=_device.U64, device=dev)
    _lib.call("nttmul_sweep_random", int(bits), int(nsamples), int(seed) & _MASK64,
              t_dev.data_ptr(), r_dev.data_ptr(), _device.stream_ptr())
    mism, key = _sweep_finish(tallies, t_dev, r_dev)
    if not mism:
        return 0, None
    s, vi = divmod(key, 3)
    lo = span = 1 << (int(bits) - 1)
    q = (lo + _splitmix_at(int(seed), 3 * s + 1) % span) | 1
    a = _splitmix_at(int(seed), 3 * s + 2) % q
    b = _splitmix_at(int(seed), 3 * s + 3) % q
    return mism, (q, a * b, vi)


def gather(x: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """out[..., v] = x[..., idx[v]] for a contiguous CUDA [n] / [batch, n] tensor."""
    op = _Operand(x, "x", False)
    batch, n = _shape(op)
    if idx.numel() != n:
        raise ValueError("index length must equal n")
    out = torch.empty_like(op.dev)
    _lib.call("nttmul_gather", out.data_ptr(), op.dev.data_ptr(), idx.data_ptr(), n, batch,
              _device.stream_ptr())
    return out
