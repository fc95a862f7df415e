"""Host logic on CPU: plan scalars, prime / root selection, modular-reduction
scalars and the C ABI surface (symbols, host-only constant preparation and
argument validation - no kernel launches)."""

from __future__ import annotations

import ctypes
import os
import random
import re

import numpy as np
import pytest

import oracle
import paper_2209_01290_b200 as nt
from paper_2209_01290_b200 import _lib
from conftest import ROOT


# ---- prime / root parity with the reference ------------------------------

def test_plan_scalars_match_reference(golden):
    for p in golden["plans"]:
        plan = nt.build_plan(p["n"], bits=p["bits"], seed=p["seed"], variant=p["variant"])
        assert (plan.q, plan.psi, plan.psi_inv, plan.omega, plan.n_inv) == \
            (p["q"], p["psi"], p["psi_inv"], p["omega"], p["n_inv"]), p
        # tw_inv[1] = psi^-(n/2) (folded into the last GS stage)
        assert plan.w1_inv == p["tw_inv_head"][1] if p["n"] >= 2 else True


def test_rns_bases_match_reference(golden):
    for g in golden["bases"]:
        basis = nt.RnsBasis.build(g["n"], g["bits"], g["k"], seed=g["seed"])
        assert list(basis.primes) == g["primes"]
        assert [p.psi for p in basis.plans] == g["psis"]
        assert str(basis.big_q) == g["big_q"]


def test_baseline_cfg3_first_prime():
    # first prime of RnsBasis.build(2^16, 60, 21, seed=0)
    assert nt.generate_prime(60, 1 << 16, 0) == 1152921504606584833


def test_is_prime_and_bit_reverse():
    assert nt.is_prime(2) and nt.is_prime(3) and not nt.is_prime(1)
    assert not nt.is_prime(3215031751)  # strong pseudoprime to bases 2,3,5,7
    assert nt.is_prime((1 << 61) - 1)
    assert [nt.bit_reverse(i, 3) for i in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]
    with pytest.raises(ValueError):
        nt.bit_reverse(8, 3)


def test_generate_prime_rejects():
    with pytest.raises(nt.ParameterError):
        nt.generate_prime(63, 16)
    with pytest.raises(nt.ParameterError):
        nt.generate_prime(30, 24)
    with pytest.raises(nt.ParameterError):
        nt.generate_prime(4, 64)


def test_build_plan_rejects():
    with pytest.raises(nt.ParameterError):
        nt.build_plan(24, bits=20)
    with pytest.raises(nt.ParameterError):
        nt.build_plan(16, 41)
    with pytest.raises(nt.ParameterError):
        nt.build_plan(16, 3 * 11 * 32 * 31 + 1)
    with pytest.raises(nt.ParameterError):
        nt.build_plan(16)
    with pytest.raises(nt.ModulusTooLargeError):
        nt.build_plan(16, bits=62, variant="dhem")


def test_plan_save_load(tmp_path):
    plan = nt.build_plan(128, bits=30, seed=2, variant="classical")
    path = tmp_path / "plan.txt"
    nt.save_plan(plan, path)
    back = nt.load_plan(path)
    assert (back.n, back.q, back.psi, back.reduction_variant) == \
        (plan.n, plan.q, plan.psi, "classical")
    path.write_text("16 97\n")
    with pytest.raises(nt.ParameterError):
        nt.load_plan(path)
    path.write_text("16 929 7 proposed\n")  # 7 is not a 32nd root of unity mod 929
    with pytest.raises(nt.ParameterError):
        nt.load_plan(path)


def test_basis_save_load_and_crt(tmp_path):
    basis = nt.RnsBasis.build(16, 28, 3, seed=3)
    path = tmp_path / "basis.txt"
    basis.save(path)
    back = nt.load_basis(path)
    assert back.primes == basis.primes and back.big_q == basis.big_q
    rng = random.Random(4)
    vals = [rng.randrange(basis.big_q) for _ in range(16)]
    assert oracle.crt_reconstruct(oracle.crt_decompose(vals, basis.primes), basis.primes) == vals
    with pytest.raises(ValueError):
        nt.decompose([basis.big_q], basis)  # range check precedes any GPU work
    ref = oracle.reference()
    if ref is not None:  # pin the CRT oracle to the reference itself
        rb = ref.RnsBasis.build(16, 28, 3, seed=3)
        assert list(rb.primes) == list(basis.primes)
        dec = ref.decompose(vals, rb)
        assert np.array_equal(np.stack(dec), oracle.crt_decompose(vals, basis.primes))
        assert ref.reconstruct(dec, rb) == oracle.crt_reconstruct(dec, basis.primes)


def test_words_conversion_roundtrip():
    rng = random.Random(9)
    for W in (1, 3, 20):
        vals = [0, 1, (1 << (64 * W)) - 1] + [rng.randrange(1 << (64 * W)) for _ in range(20)]
        words = nt.ints_to_words(vals, W)
        assert words.shape == (len(vals), W) and words.dtype == np.uint64
        assert nt.words_to_ints(words) == vals
    plan = nt.build_plan(8, bits=20, seed=0)
    with pytest.raises(nt.ParameterError):
        nt.RnsBasis.from_plans([plan, plan])


def test_workload_size():
    assert nt.workload_size(1240, 28) == 45
    assert nt.workload_size(1240, 30) == 42
    assert nt.workload_size(61, 30) == 3
    with pytest.raises(ValueError):
        nt.workload_size(0, 30)


# ---- modular arithmetic scalars (reference modarith semantics) -----------

def test_named_triple(golden):
    t = golden["named_triple"]
    mod = nt.Modulus(t["q"])
    x = t["a"] * t["b"]
    for fn in (nt.barrett_classical, nt.barrett_dhem, nt.barrett_proposed):
        assert fn(x, mod) == t["want"] == 30439
    s = nt.ReductionStats()
    nt.barrett_classical(x, mod, s)
    assert s.subtractions_2 == 1  # the classical variant's second subtraction
    s = nt.ReductionStats()
    nt.barrett_proposed(x, mod, s)
    assert s.subtractions_2 == 0


def test_exhaustive_tiny_moduli():
    for q in range(3, 64, 2):
        mod = nt.Modulus(q)
        for x in range(q * q):
            assert nt.barrett_classical(x, mod) == nt.barrett_dhem(x, mod) == \
                nt.barrett_proposed(x, mod) == x % q


def test_modulus_constants_and_errors():
    q = (1 << 62) - 57
    mod = nt.Modulus(q)
    assert mod.m == 62 and mod.mu_dhem is None
    assert mod.mu_proposed == (1 << 125) // q
    with pytest.raises(ValueError):
        nt.Modulus(4)
    with pytest.raises(nt.ModulusTooLargeError):
        nt.Modulus((1 << 63) - 25)
    with pytest.raises(nt.ModulusTooLargeError):
        mod.reduction_params("dhem")
    assert nt.half_mod(5, nt.Modulus(13)) == 5 * 7 % 13
    assert nt.mod_add(12, 5, nt.Modulus(13)) == 4 and nt.mod_sub(2, 5, nt.Modulus(13)) == 10


def test_fused_butterfly_scalar():
    mod = nt.Modulus(12289)
    rng = random.Random(8)
    ctr = nt.OpCounter()
    for _ in range(50):
        a0, a1, b0, b1 = (rng.randrange(mod.q) for _ in range(4))
        al = rng.randrange(1, mod.q)
        c0, c1 = nt.fused_butterfly(a0, a1, b0, b1, al, mod, ctr)
        assert c0 == (a0 * b0 + al * a1 * b1) % mod.q
        assert c1 == (a0 * b1 + a1 * b0) % mod.q
    assert (ctr.modmul, ctr.modadd_sub) == (200, 250)


# ---- C ABI ------------------------------------------------------------------

def _declared_functions():
    with open(os.path.join(ROOT, "include", "nttmul_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(nttmul_\w+)\s*\(", text,
                                 re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)
    assert lib.nttmul_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a():
    """The shipped cubin targets sm_100a (cuobjdump, no GPU needed)."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_limb_prepare_host_only():
    plan = nt.build_plan(1 << 16, bits=60, seed=0)
    limb = plan.limb()
    q = plan.q
    mode, mu, s_in, s_out = plan.mod.reduction_params("proposed")
    assert limb.q == q and limb.mode == mode and limb.s_in == s_in
    # quot = umulhi(c, mu_sh) >> s_hi == (c * mu) >> s_out for all c
    rng = random.Random(1)
    for _ in range(1000):
        c = rng.randrange(1 << (plan.mod.m + 2))
        assert ((c * limb.mu_sh) >> 64) >> limb.s_hi == (c * mu) >> s_out
    f_full = pow(plan.n, -1, q)
    f_skip = pow(plan.n // 2, -1, q)
    assert list(limb.sc_full) == [f_full, (f_full << 64) // q, plan.w1_inv * f_full % q,
                                  ((plan.w1_inv * f_full % q) << 64) // q]
    assert limb.sc_skip[0] == f_skip
    for variant in ("classical", "dhem", "builtin"):
        lb = nt.build_plan(256, bits=30, seed=0, variant=variant).limb()
        assert lb.mode == {"classical": 1, "dhem": 2, "builtin": 0}[variant]


def test_abi_rejects_bad_arguments_without_launching():
    lib = _lib.load()
    limb = _lib.LimbStruct()
    assert lib.nttmul_limb_prepare(ctypes.byref(limb), 4, 2, 1, 0, 3, 4, 1) == 1  # even q
    assert lib.nttmul_limb_prepare(ctypes.byref(limb), (1 << 63) + 1, 2, 1, 0, 3, 4, 1) == 1
    assert lib.nttmul_limb_prepare(ctypes.byref(limb), 97, 7, 1, 0, 3, 4, 1) == 1  # mode
    assert b"mode" in lib.nttmul_last_error()
    # log_n out of range is rejected before any pointer is touched
    assert lib.nttmul_ntt_ct(None, None, 97, 2, 1, 5, 10, 0, 0, 1, None) == 1
    assert lib.nttmul_ntt_ct(None, None, 97, 2, 1, 5, 10, 0, 18, 1, None) == 1
    # empty batch is a no-op
    assert lib.nttmul_ntt_ct(None, None, 97, 2, 1, 5, 10, 0, 4, 0, None) == 0
    # half_q must be (q+1)/2
    assert lib.nttmul_intt_gs(None, None, 97, 50, 2, 1, 5, 10, 1, 0, 4, 1, 1, None) == 1
    # host (non-device) pointers are refused, not dereferenced
    buf = np.zeros(16, dtype=np.uint64)
    st = lib.nttmul_hadamard(buf.ctypes.data, buf.ctypes.data, buf.ctypes.data, 16, 97, 2, 1,
                             5, 10, None)
    assert st in (3, 5)


def test_product_path_has_no_oracle_import():
    """The package never imports oracle/ (the checker) or any CPU kernel twin."""
    pkg = os.path.join(ROOT, "paper_2209_01290_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
            assert "_kernels_py" not in src, f


# ---- device arithmetic restated on the host (error bounds of shoup4) -------

def _shoup4_host(x: int, w: int, wp: int, q: int) -> int:
    """Bit-exact host model of modarith.cuh shoup4 (3-partial-product quotient)."""
    M32, M64 = (1 << 32) - 1, (1 << 64) - 1
    xl, xh, wpl, wph = x & M32, x >> 32, wp & M32, wp >> 32
    b, c = xl * wph, xh * wpl
    qh = (xh * wph + (b >> 32) + (c >> 32)) & M64
    nq = (1 << 64) - q
    a = (xl * (w & M32) + (qh & M32) * (nq & M32)) & M64
    h = ((a >> 32) + xl * (w >> 32) + xh * (w & M32) + (qh & M32) * (nq >> 32)
         + (qh >> 32) * (nq & M32)) & M32
    return (h << 32) | (a & M32)


@pytest.mark.parametrize("bits", [20, 30, 59, 60, 61, 62])
def test_shoup4_bound_and_congruence(bits):
    rng = random.Random(bits)
    for _ in range(4000):
        q = rng.randrange(1 << (bits - 1), 1 << bits) | 1
        w = rng.randrange(q)
        wp = (w << 64) // q
        # inputs up to the largest lazy value the kernels feed in: 8q (q < 2^61)
        # or 4q (62-bit moduli), plus the extremes
        top = min((8 if bits <= 61 else 4) * q, 1 << 64)
        for x in (0, 1, top - 1, rng.randrange(top), rng.randrange(1 << 64)):
            r = _shoup4_host(x, w, wp, q)
            assert r < 4 * q
            assert r % q == x * w % q


def test_mixed_variant_basis_accepted():
    """The reference's RnsBasis.from_plans accepts plans of different
    reduction variants (rns.py:61-73); the device launch then runs every limb
    with one variant (identical canonical residues)."""
    n = 1 << 13
    primes = nt.RnsBasis.build(n, 60, 3, seed=0).primes
    mixed = nt.RnsBasis.from_plans([nt.build_plan(n, q, seed=0, variant=v)
                                    for q, v in zip(primes, ["classical", "dhem", "builtin"])])
    assert mixed.device_variant == "proposed"
    assert mixed.mode & 0xFF == 2  # the proposed variant's one-subtraction mode
    same = nt.RnsBasis.from_plans([nt.build_plan(n, q, seed=0, variant="classical")
                                   for q in primes])
    assert same.device_variant == "classical" and same.mode & 0xFF == 1

