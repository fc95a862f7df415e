"""Pin the C oracle (oracle/ntt_oracle.c) to the reference's own outputs.

Every vector below was produced by the unmodified reference package
(tests/golden/make_golden.py).  CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import digest, rand


def _cases(golden):
    return {c["key"]: c for c in golden["vector_cases"]}


def test_twiddle_tables_match_reference(golden):
    for p in golden["plans"]:
        if p["n"] > (1 << 14):
            continue
        f, v = oracle.twiddles(p["q"], p["psi"], p["n"].bit_length() - 1)
        assert digest(f) == p["tw_fwd_sha"], p
        assert digest(v) == p["tw_inv_sha"], p


def test_spec_example_table():
    # n=4, q=13, psi=5 -> tw_fwd = [1, 12, 5, 8]
    f, _ = oracle.twiddles(13, 5, 2)
    assert f.tolist() == [1, 12, 5, 8]


@pytest.mark.parametrize("variant", ["proposed", "classical", "builtin"])
def test_small_vectors_every_op(golden, vectors, variant):
    for key, c in _cases(golden).items():
        n, q = c["n"], c["q"]
        if variant == "classical" and q.bit_length() > 62:
            continue
        f, v = oracle.twiddles(q, c["psi"], n.bit_length() - 1)
        red = oracle.reduction_params(q, variant)
        a, b, x = vectors[key + "_a"], vectors[key + "_b"], vectors[key + "_x"]

        t = a.copy()
        cnt = np.zeros(5, dtype=np.uint64)
        oracle.ntt_ct(t, f, q, *red, False, cnt)
        assert np.array_equal(t, vectors[key + "_ntt"]), key
        assert cnt.tolist() == c["ntt_counts"][:2] + [0] + c["ntt_counts"][3:4] + [0]

        t = x.copy()
        oracle.intt_gs(t, v, q, (q + 1) // 2, *red, False, False)
        assert np.array_equal(t, vectors[key + "_intt"]), key
        t = x.copy()
        cnt = np.zeros(5, dtype=np.uint64)
        oracle.intt_gs(t, v, q, (q + 1) // 2, *red, True, False, cnt)
        assert np.array_equal(t, vectors[key + "_intts"]), key
        assert cnt.tolist() == c["intts_counts"]

        if n >= 4:
            t = a.copy()
            oracle.ntt_ct(t, f, q, *red, True)
            assert np.array_equal(t, vectors[key + "_nttt"]), key
            t = x.copy()
            oracle.intt_gs(t, v, q, (q + 1) // 2, *red, True, True)
            assert np.array_equal(t, vectors[key + "_inttt"]), key
            ah, bh = a.copy(), b.copy()
            oracle.ntt_ct(ah, f, q, *red, True)
            oracle.ntt_ct(bh, f, q, *red, True)
            ch = np.empty(n, dtype=np.uint64)
            cnt = np.zeros(5, dtype=np.uint64)
            oracle.fused_middle(ah, bh, ch, f, q, *red, cnt)
            assert np.array_equal(ch, vectors[key + "_mid"]), key
            assert cnt.tolist() == c["mid_counts"]
            cnt = np.zeros(5, dtype=np.uint64)
            got = oracle.polymul_fused(a, b, q, c["psi"], variant, counts=cnt)
            assert np.array_equal(got, vectors[key + "_fused"]), key
            assert cnt.tolist() == c["fused_counts"]

        out = np.empty(n, dtype=np.uint64)
        oracle.hadamard(a, b, out, q, *red)
        assert np.array_equal(out, vectors[key + "_had"]), key
        t = a.copy()
        oracle.scale(t, c["scale_factor"], q, *red)
        assert np.array_equal(t, vectors[key + "_scale"]), key
        if n <= 1024:
            assert np.array_equal(oracle.negacyclic_naive(a, b, q), vectors[key + "_naive"])


def test_fused_equals_naive(golden, vectors):
    for key, c in _cases(golden).items():
        if c["n"] >= 4 and c["n"] <= 1024:
            assert np.array_equal(vectors[key + "_fused"], vectors[key + "_naive"]), key


@pytest.mark.parametrize("log_n", [12, 13, 14, 15, 16, 17])
def test_large_digests(golden, log_n):
    rec = next(r for r in golden["large"] if r["n"] == 1 << log_n)
    q, psi, n = rec["q"], rec["psi"], rec["n"]
    f, v = oracle.twiddles(q, psi, log_n)
    red = oracle.reduction_params(q)
    a, b = rand(q, n, rec["a_seed"]), rand(q, n, rec["b_seed"])
    t = a.copy()
    oracle.ntt_ct(t, f, q, *red, False)
    assert digest(t) == rec["ntt_sha"]
    t = a.copy()
    oracle.ntt_ct(t, f, q, *red, True)
    assert digest(t) == rec["nttt_sha"]
    t = rand(q, n, rec["intt_x_seed"])
    oracle.intt_gs(t, v, q, (q + 1) // 2, *red, False, False)
    assert digest(t) == rec["intt_sha"]
    cnt = np.zeros(5, dtype=np.uint64)
    c = oracle.polymul_fused(a, b, q, psi, counts=cnt, tables=(f, v))
    assert digest(c) == rec["fused_sha"]
    assert cnt.tolist() == rec["fused_counts"]


def test_mulmod_loop_sinks(golden):
    for s in golden["mulmod_loop"]:
        q = s["q"]
        a, b = rand(q, s["n"], s["a_seed"]), rand(q, s["n"], s["b_seed"])
        red = oracle.reduction_params(q, s["variant"])
        assert oracle.mulmod_loop(a, b, q, *red, s["passes"]) == s["sink"]


def test_named_triple_every_variant(golden):
    t = golden["named_triple"]
    q = t["q"]
    for variant in ("builtin", "classical", "dhem", "proposed"):
        out = np.empty(1, dtype=np.uint64)
        oracle.hadamard(np.array([t["a"]], np.uint64), np.array([t["b"]], np.uint64), out,
                        q, *oracle.reduction_params(q, variant))
        assert int(out[0]) == t["want"] == 30439


def test_reference_package_agrees_when_present():
    """If oracle/_ref (the real reference) is built here, cross-check directly."""
    nt = oracle.reference()
    if nt is None:
        pytest.skip("oracle/_ref not built")
    plan = nt.build_plan(1 << 10, bits=62, seed=7)
    a, b = rand(plan.q, plan.n, 1), rand(plan.q, plan.n, 2)
    want = nt.polymul_fused(nt.Polynomial(a.copy()), nt.Polynomial(b.copy()), plan)
    assert np.array_equal(oracle.polymul_fused(a, b, plan.q, plan.psi), want)
