"""Transform plans (reference pkg/src/nttmul/params.py).

Host side (Python ints, off the timed path): the deterministic NTT-prime
scan and the seeded primitive-root search.  Both must select exactly the
reference's (q, psi) - twiddle tables and therefore ``ntt_ct`` outputs depend
on psi - so they follow the reference algorithm step for step:

* ``generate_prime`` (params.py:61-85): candidates q = 2n*k + 1, k scanned
  downward from the top of the bit range, the start rotated by
  ``seed % count``; first prime wins.
* ``find_primitive_root`` (params.py:88-103): ``random.Random(seed)`` draws
  g in [2, q-2]; psi = g^((q-1)/2n) is accepted iff psi^n == q-1.

Device side: the twiddle tables tw_fwd[i] = psi^br(i) and
tw_inv[i] = psi^-br(i) (params.py:157-167) are generated ON THE GPU
(``nttmul_twiddle_tables``), together with the {w, floor(w 2^64/q)} pair
tables the kernels read.  A plan built without a GPU keeps its scalars and
materialises its tables on first device use.
"""

from __future__ import annotations

import random

import torch

from . import _device, _lib
from .modarith import WORD_SIZE, Modulus

# Deterministic Miller-Rabin bases for n < 3.3e24 (covers 64-bit).
_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


class ParameterError(ValueError):
    """Invalid or inconsistent transform parameters."""


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for 64-bit integers."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    r = ((n - 1) & -(n - 1)).bit_length() - 1
    d = (n - 1) >> r
    for a in _MR_BASES:
        y = pow(a, d, n)
        if y in (1, n - 1):
            continue
        for _ in range(r - 1):
            y = y * y % n
            if y == n - 1:
                break
        else:
            return False
    return True


def bit_reverse(i: int, bits: int) -> int:
    """Reverse the low ``bits`` bits of i."""
    if not 0 <= i < (1 << bits):
        raise ValueError(f"index {i} out of range for {bits} bits")
    return int(format(i, f"0{bits}b")[::-1], 2) if bits else 0


def _check_n(n: int) -> None:
    if n < 2 or n & (n - 1):
        raise ParameterError(f"n must be a power of two >= 2, got {n}")


def generate_prime(bits: int, n: int, seed: int = 0) -> int:
    """The reference's deterministic ``bits``-bit prime with q = 1 mod 2n."""
    if not 4 <= bits <= WORD_SIZE - 2:
        raise ParameterError(f"bits must be in [4, {WORD_SIZE - 2}], got {bits}")
    _check_n(n)
    step = 2 * n
    if step >= 1 << bits:
        raise ParameterError(f"2n = {step} leaves no {bits}-bit candidates")
    hi = ((1 << bits) - 2) // step            # largest k with q < 2^bits
    lo = ((1 << (bits - 1)) - 1) // step + 1  # smallest k with q >= 2^(bits-1)
    if lo > hi:
        raise ParameterError(f"no {bits}-bit candidates with q = 1 mod {step}")
    count = hi - lo + 1
    start = seed % count
    for t in range(count):
        q = step * (hi - (start + t) % count) + 1
        if is_prime(q):
            return q
    raise ParameterError(f"no {bits}-bit prime with q = 1 mod {step}")


def find_primitive_root(q: int, two_n: int, seed: int = 0) -> int:
    """The reference's seeded choice of a primitive 2n-th root of unity."""
    if (q - 1) % two_n:
        raise ParameterError(f"{two_n} does not divide q - 1 = {q - 1}")
    rng = random.Random(seed)
    e = (q - 1) // two_n
    while True:
        psi = pow(rng.randrange(2, q - 1), e, q)
        if pow(psi, two_n // 2, q) == q - 1:
            return psi


class NttPlan:
    """Everything the transforms of one (n, q) need.

    Scalars mirror the reference NttPlan (params.py:106-127).  ``tw_fwd`` /
    ``tw_inv`` are CUDA uint64[n] tensors in the reference layout; the kernels
    read ``fwd_pairs`` / ``inv_pairs`` (uint64[n, 2]: value, Shoup companion).
    """

    def __init__(self, n: int, log_n: int, mod: Modulus, psi: int, psi_inv: int,
                 omega: int, n_inv: int, tw_fwd=None, tw_inv=None,
                 reduction_variant: str = "proposed"):
        self.n, self.log_n, self.mod = n, log_n, mod
        self.psi, self.psi_inv, self.omega, self.n_inv = psi, psi_inv, omega, n_inv
        self.reduction_variant = reduction_variant
        # explicit tables (possibly corrupted, for validate_plan) as given;
        # None -> generated on the device from psi
        self._tw_src = None if tw_fwd is None else (_device.to_device(tw_fwd),
                                                    _device.to_device(tw_inv))
        # per CUDA device: (tw_fwd, tw_inv, fwd_pairs, inv_pairs, limb bytes)
        self._dev_tables: dict = {}
        self._cache: dict = {}

    # -- scalars ----------------------------------------------------------
    @property
    def q(self) -> int:
        return self.mod.q

    @property
    def red_args(self) -> tuple[int, int, int, int, int]:
        """(q, mode, mu, s_in, s_out) for this plan's variant."""
        return (self.q, *self.mod.reduction_params(self.reduction_variant))

    @property
    def w1_inv(self) -> int:
        """tw_inv[1] = psi^-(n/2) (the last GS stage's twiddle)."""
        return pow(self.psi_inv, self.n // 2, self.q) if self.n >= 2 else 1

    # -- device tables (one set per CUDA device) ---------------------------
    def _tables(self) -> tuple:
        t = self._dev_tables.get(_device.index())
        if t is not None:
            return t
        dev = _device.device()
        st = _device.stream_ptr()
        n = self.n
        fwd_pairs = torch.empty((n, 2), dtype=_device.U64, device=dev)
        inv_pairs = torch.empty((n, 2), dtype=_device.U64, device=dev)
        if self._tw_src is None:
            tw_fwd = torch.empty(n, dtype=_device.U64, device=dev)
            tw_inv = torch.empty(n, dtype=_device.U64, device=dev)
            _lib.call("nttmul_twiddle_tables", tw_fwd.data_ptr(), tw_inv.data_ptr(),
                      fwd_pairs.data_ptr(), inv_pairs.data_ptr(), self.q, self.psi,
                      self.psi_inv, self.log_n, st)
        else:  # explicit (possibly corrupted) tables: pair them as given
            tw_fwd, tw_inv = (x.to(dev) for x in self._tw_src)
            _lib.call("nttmul_shoup_pairs", fwd_pairs.data_ptr(), tw_fwd.data_ptr(),
                      self.q, n, st)
            _lib.call("nttmul_shoup_pairs", inv_pairs.data_ptr(), tw_inv.data_ptr(),
                      self.q, n, st)
        raw = bytes(self.limb())
        limb = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
        t = (tw_fwd, tw_inv, fwd_pairs, inv_pairs, limb)
        self._dev_tables[dev.index] = t
        from . import kernels

        kernels.register_pairs(tw_fwd, fwd_pairs, self.q, w1=1)
        kernels.register_pairs(tw_inv, inv_pairs, self.q, w1=self.w1_inv)
        return t

    @property
    def tables_ready(self) -> bool:
        return torch.cuda.is_available() and \
            torch.cuda.current_device() in self._dev_tables

    @property
    def tw_fwd(self) -> torch.Tensor:
        return self._tables()[0]

    @property
    def tw_inv(self) -> torch.Tensor:
        return self._tables()[1]

    @property
    def fwd_pairs(self) -> torch.Tensor:
        return self._tables()[2]

    @property
    def inv_pairs(self) -> torch.Tensor:
        return self._tables()[3]

    def limb(self) -> "_lib.LimbStruct":
        """Host nttmul_limb_t for this plan."""
        q, mode, mu, s_in, s_out = self.red_args
        return _lib.prepare_limb(q, mode, mu, s_in, s_out, self.log_n, self.w1_inv)

    def limb_device(self) -> torch.Tensor:
        """Device copy of :meth:`limb` (96 bytes) on the current device."""
        return self._tables()[4]

    def __repr__(self) -> str:
        return (f"NttPlan(n={self.n}, q={self.q}, psi={self.psi}, "
                f"variant={self.reduction_variant!r})")


def build_plan(n: int, q: int | None = None, *, bits: int | None = None,
               seed: int = 0, variant: str = "proposed") -> NttPlan:
    """Build and validate a plan; q given directly or generated from (bits, seed)."""
    _check_n(n)
    if q is None:
        if bits is None:
            raise ParameterError("either q or bits must be given")
        q = generate_prime(bits, n, seed)
    if not is_prime(q):
        raise ParameterError(f"q = {q} is not prime")
    if (q - 1) % (2 * n):
        raise ParameterError(f"2n = {2 * n} does not divide q - 1")
    mod = Modulus(q)
    mod.reduction_params(variant)  # reject an inadmissible variant early
    return _plan_from_root(n, mod, find_primitive_root(q, 2 * n, seed), variant)


def _plan_from_root(n: int, mod: Modulus, psi: int, variant: str) -> NttPlan:
    q = mod.q
    psi_inv = pow(psi, q - 2, q)
    plan = NttPlan(n=n, log_n=n.bit_length() - 1, mod=mod, psi=psi, psi_inv=psi_inv,
                   omega=psi * psi % q, n_inv=pow(n, q - 2, q), reduction_variant=variant)
    validate_plan(plan, tables=torch.cuda.is_available())
    return plan


def validate_plan(plan: NttPlan, tables: bool | None = None) -> None:
    """Check every structural invariant; ParameterError on corruption.

    The twiddle tables are checked on the device (``nttmul_check_twiddles``)
    when they exist (or ``tables=True``); scalar invariants always.
    """
    n, q = plan.n, plan.q
    if n < 2 or n != 1 << plan.log_n:
        raise ParameterError("n is not a power of two >= 2")
    if not is_prime(q):
        raise ParameterError(f"q = {q} failed the primality test")
    if (q - 1) % (2 * n):
        raise ParameterError("2n does not divide q - 1")
    if pow(plan.psi, n, q) != q - 1 or pow(plan.psi, 2 * n, q) != 1:
        raise ParameterError("psi is not a primitive 2n-th root of unity")
    if plan.psi * plan.psi_inv % q != 1:
        raise ParameterError("psi_inv is not the inverse of psi")
    if n % q * plan.n_inv % q != 1:
        raise ParameterError("n_inv is not the inverse of n")
    if plan.omega != plan.psi * plan.psi % q:
        raise ParameterError("omega is not psi^2")
    if tables is None:
        tables = plan._tw_src is not None
    if not tables:
        return
    f, v = plan.tw_fwd, plan.tw_inv
    if f.numel() != n or v.numel() != n:
        raise ParameterError("twiddle tables have the wrong length")
    bad = torch.zeros(1, dtype=_device.U64, device=f.device)
    _lib.call("nttmul_check_twiddles", f.data_ptr(), v.data_ptr(), q, n, bad.data_ptr(),
              _device.stream_ptr())
    nbad = int(bad.item())
    if nbad:
        raise ParameterError(f"{nbad} twiddle entries are not inverse pairs (or tw[0] != 1)")


def save_plan(plan: NttPlan, path) -> None:
    """Write the one-line header ``n q psi variant``."""
    with open(path, "w") as fh:
        fh.write(f"{plan.n} {plan.q} {plan.psi} {plan.reduction_variant}\n")


def load_plan(path) -> NttPlan:
    """Rebuild and validate a plan from its header line."""
    with open(path) as fh:
        fields = fh.readline().split()
    if len(fields) != 4:
        raise ParameterError(f"{path}: expected header 'n q psi variant'")
    try:
        n, q, psi = (int(x) for x in fields[:3])
    except ValueError as exc:
        raise ParameterError(f"{path}: malformed header: {exc}") from None
    if n < 2 or n & (n - 1):
        raise ParameterError(f"{path}: n must be a power of two >= 2")
    if not is_prime(q):
        raise ParameterError(f"{path}: q = {q} is not prime")
    if (q - 1) % (2 * n):
        raise ParameterError(f"{path}: 2n does not divide q - 1")
    mod = Modulus(q)
    mod.reduction_params(fields[3])
    return _plan_from_root(n, mod, psi, fields[3])


def _limb_array(limbs) -> torch.Tensor:
    """Pack host LimbStructs into one device byte tensor [L * 96]."""
    raw = b"".join(bytes(lb) for lb in limbs)
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(_device.device())


__all__ = ["ParameterError", "NttPlan", "bit_reverse", "build_plan", "find_primitive_root",
           "generate_prime", "is_prime", "load_plan", "save_plan", "validate_plan"]
