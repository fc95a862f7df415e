"""CPU check of the lazy-reduction bounds the sm_100a kernels rely on
(paper_2209_01290_b200/csrc/modarith.cuh): a bit-level restatement of
``mulhi_approx``, ``shoup4`` and ``mulred_lazy`` in Python integers, driven
with random and extreme operands for the BASELINE primes and small moduli.
The GPU parity tests exercise the CUDA code itself; this pins the arithmetic
argument (quotient undershoot, output ranges) independently of a GPU."""

from __future__ import annotations

import random

import pytest

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1


def lo(x):
    return x & M32


def hi(x):
    return (x >> 32) & M32


def mulhi_approx(x, y):
    b = lo(x) * hi(y)
    c = hi(x) * lo(y) + lo(b)
    assert c <= M64
    r = hi(x) * hi(y) + hi(b) + hi(c)
    assert r <= M64
    return r


def shoup4(x, w, wp, q):
    b, c = lo(x) * hi(wp), hi(x) * lo(wp)
    qh = hi(x) * hi(wp) + hi(b) + hi(c)
    nq = (-q) & M64
    a = (lo(qh) * lo(nq) + lo(x) * lo(w)) & M64
    h = hi(a)
    for p in (lo(x) * hi(w), hi(x) * lo(w), lo(qh) * hi(nq), hi(qh) * lo(nq)):
        h = (p + h) & M32
    return (h << 32) | lo(a)


def limb_consts(q, variant):
    """(mu_sh, s_in, s_hi) as nttmul_limb_prepare builds them for mode 2."""
    m = q.bit_length()
    mu, s_in, s_out = {"proposed": ((1 << (2 * m + 1)) // q, m - 2, m + 3),
                       "dhem": ((1 << (2 * m + 3)) // q, m - 2, m + 5)}[variant]
    if s_out <= 64:
        return mu << (64 - s_out), s_in, 0
    return mu, s_in, s_out - 64


def mulred_lazy(a, b, q, mu_sh, s_in, s_hi):
    t = a * b
    c = t >> s_in
    assert c <= M64
    quot = mulhi_approx(c, mu_sh) >> s_hi
    return (t - quot * q) & M64


PRIMES = [1009, 998244353, 576460752303816705 + 0, 1152921504606830593,
          1152921504606584833]


@pytest.mark.parametrize("q", PRIMES)
def test_mulhi_approx_undershoot_at_most_one(q):
    rng = random.Random(q)
    for _ in range(20000):
        x, y = rng.randrange(1 << 64), rng.randrange(1 << 64)
        exact = (x * y) >> 64
        assert exact - 1 <= mulhi_approx(x, y) <= exact
    assert mulhi_approx(M64, M64) in ((M64 * M64) >> 64, ((M64 * M64) >> 64) - 1)


@pytest.mark.parametrize("q", PRIMES)
def test_shoup4_range(q):
    rng = random.Random(q + 1)
    for _ in range(20000):
        w = rng.randrange(q)
        wp = (w << 64) // q
        x = rng.choice([rng.randrange(1 << 64), rng.randrange(16 * q), M64, 0])
        r = shoup4(x, w, wp, q)
        assert r % q == x * w % q and r < 4 * q


@pytest.mark.parametrize("variant", ["proposed", "dhem"])
@pytest.mark.parametrize("q", [p for p in PRIMES if p.bit_length() <= 60])
def test_mulred_lazy_range(q, variant):
    mu_sh, s_in, s_hi = limb_consts(q, variant)
    rng = random.Random(q + 2)
    edge = [0, 1, q - 1, q, 2 * q - 1]
    for _ in range(20000):
        a = rng.choice(edge + [rng.randrange(2 * q)])
        b = rng.choice(edge + [rng.randrange(2 * q)])
        r = mulred_lazy(a, b, q, mu_sh, s_in, s_hi)
        assert r % q == a * b % q and r < 5 * q


def make_fastred(q):
    """modarith.cuh make_fastred: (r, s, ok) with r = floor(2^(64+s) / q) - 1
    computed through a double division like the device code."""
    import math

    m = q.bit_length()
    if not 35 <= m <= 62:
        return 0, 0, False
    s = m - 33
    rd = math.ldexp(1.0, 64 + s) / float(q)
    return int(rd) - 1, s, True


def reduce2q(x, q, r, s):
    k = ((x >> 32) * r >> 32) >> s
    return (x - k * q) & M64


@pytest.mark.parametrize("q", [(1 << 34) + 1, (1 << 35) - 31, 998244353 * 64 + 1,
                               576460752303816705, 1152921504606830593,
                               1152921504606584833, (1 << 62) - 57])
def test_reduce2q_range(q):
    """Multiply-based partial reduction: x - k q in [0, 2q) for any x < 2^64
    (the fused middle's inputs < 16q and outputs < 15q included)."""
    r, s, ok = make_fastred(q)
    if q.bit_length() < 35:
        assert not ok
        return
    assert ok and r < (1 << 32)
    rng = random.Random(q)
    for _ in range(50000):
        x = rng.choice([rng.randrange(1 << 64), rng.randrange(16 * q) if 16 * q < (1 << 64)
                        else rng.randrange(1 << 64), M64, 0, q - 1, q, 2 * q - 1, 2 * q])
        y = reduce2q(x, q, r, s)
        assert y % q == x % q and y < 2 * q, (x, y)
