"""GPU parity: every sm_100a entry point vs the reference (golden vectors from
the unmodified reference) and the C oracle.  Bit-exact throughout - this is
integer work, there is no tolerance.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from conftest import digest, rand

pytestmark = pytest.mark.gpu

nt = pytest.importorskip("paper_2209_01290_b200")
K = nt.kernels


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64)).cuda()


def host(t):
    return t.cpu().numpy()


def _plan(c, variant="proposed"):
    return nt.build_plan(c["n"], bits=c["bits"], seed=0, variant=variant)


# ---- plans ---------------------------------------------------------------

def test_device_twiddle_tables_match_reference(golden):
    for p in golden["plans"]:
        plan = nt.build_plan(p["n"], bits=p["bits"], seed=p["seed"], variant=p["variant"])
        assert (plan.q, plan.psi) == (p["q"], p["psi"])
        assert digest(host(plan.tw_fwd)) == p["tw_fwd_sha"]
        assert digest(host(plan.tw_inv)) == p["tw_inv_sha"]
        nt.validate_plan(plan, tables=True)


def test_validate_plan_catches_corrupted_table():
    plan = nt.build_plan(16, bits=12, seed=0)
    f = host(plan.tw_fwd).copy()
    f[5] ^= 1
    bad = nt.NttPlan(n=plan.n, log_n=plan.log_n, mod=plan.mod, psi=plan.psi,
                     psi_inv=plan.psi_inv, omega=plan.omega, n_inv=plan.n_inv,
                     tw_fwd=f, tw_inv=host(plan.tw_inv))
    with pytest.raises(nt.ParameterError):
        nt.validate_plan(bad)


# ---- kernel surface on the reference's own vectors ---------------------

@pytest.mark.parametrize("variant", ["proposed", "classical", "builtin", "dhem"])
def test_kernel_surface_small_vectors(golden, vectors, variant):
    for c in golden["vector_cases"]:
        key, n, q = c["key"], c["n"], c["q"]
        if variant == "dhem" and q.bit_length() > 60:
            continue
        plan = _plan(c, variant)
        red = plan.red_args
        a, b, x = vectors[key + "_a"], vectors[key + "_b"], vectors[key + "_x"]

        t = dev(a)
        cnt = np.zeros(5, dtype=np.uint64)
        K.ntt_ct(t, plan.tw_fwd, *red, False, cnt)
        assert np.array_equal(host(t), vectors[key + "_ntt"]), key
        assert cnt.tolist() == c["ntt_counts"][:2] + [0, c["ntt_counts"][3], 0]

        t = dev(x)
        cnt = np.zeros(5, dtype=np.uint64)
        K.intt_gs(t, plan.tw_inv, q, (q + 1) // 2, *red[1:], False, False, cnt)
        assert np.array_equal(host(t), vectors[key + "_intt"]), key
        assert cnt.tolist() == c["intt_counts"]
        t = dev(x)
        cnt = np.zeros(5, dtype=np.uint64)
        K.intt_gs(t, plan.tw_inv, q, (q + 1) // 2, *red[1:], True, False, cnt)
        assert np.array_equal(host(t), vectors[key + "_intts"]), key
        assert cnt.tolist() == c["intts_counts"]

        if n >= 4:
            t = dev(a)
            K.ntt_ct(t, plan.tw_fwd, *red, True)
            assert np.array_equal(host(t), vectors[key + "_nttt"]), key
            t = dev(x)
            K.intt_gs(t, plan.tw_inv, q, (q + 1) // 2, *red[1:], True, True)
            assert np.array_equal(host(t), vectors[key + "_inttt"]), key
            ah, bh = dev(a), dev(b)
            K.ntt_ct(ah, plan.tw_fwd, *red, True)
            K.ntt_ct(bh, plan.tw_fwd, *red, True)
            ch = torch.empty_like(ah)
            cnt = np.zeros(5, dtype=np.uint64)
            K.fused_middle(ah, bh, ch, plan.tw_fwd, *red, cnt)
            assert np.array_equal(host(ch), vectors[key + "_mid"]), key
            assert cnt.tolist() == c["mid_counts"]

        out = torch.empty(n, dtype=torch.uint64, device="cuda")
        K.hadamard(dev(a), dev(b), out, *red)
        assert np.array_equal(host(out), vectors[key + "_had"]), key
        t = dev(a)
        K.scale(t, c["scale_factor"], *red)
        assert np.array_equal(host(t), vectors[key + "_scale"]), key


def test_kernel_surface_numpy_host_buffers(golden, vectors):
    """numpy operands: staged to HBM and written back in place (drop-in)."""
    c = next(c for c in golden["vector_cases"] if c["n"] == 4096)
    plan = _plan(c)
    t = vectors[c["key"] + "_a"].copy()
    tw = host(plan.tw_fwd)
    K.ntt_ct(t, tw, *plan.red_args, False, None)
    assert np.array_equal(t, vectors[c["key"] + "_ntt"])
    with pytest.raises(ValueError):
        K.ntt_ct(t.astype(np.int64), tw, *plan.red_args, False, None)
    with pytest.raises(TypeError):
        K.ntt_ct([1, 2, 3, 4], tw, *plan.red_args, False, None)


def test_public_api_small_vectors(golden, vectors):
    for c in golden["vector_cases"]:
        key, n = c["key"], c["n"]
        plan = _plan(c)
        a, b = vectors[key + "_a"], vectors[key + "_b"]
        ctr = nt.OpCounter()
        got = nt.polymul_fused(a, b, plan, ctr)
        assert isinstance(got, np.ndarray)
        assert np.array_equal(got, vectors[key + "_fused"]), key
        assert list(ctr.as_tuple()) == c["fused_counts"], key
        ctr = nt.OpCounter()
        got = nt.polymul_ntt(dev(a), dev(b), plan, ctr)
        assert np.array_equal(host(got), vectors[key + "_pntt"]), key
        assert list(ctr.as_tuple()) == c["pntt_counts"], key
        p = nt.Polynomial(a)
        ctr = nt.OpCounter()
        nt.ntt_ct(p, plan, ctr)
        assert p.ordering == "bit_reversed"
        assert np.array_equal(p.numpy(), vectors[key + "_ntt"])
        nt.intt_gs_scaled(p, plan)
        assert np.array_equal(p.numpy(), a)
        assert np.array_equal(nt.hadamard(a, b, plan), vectors[key + "_had"])


@pytest.mark.parametrize("log_n", [12, 13, 14, 15, 16, 17])
def test_large_sizes_match_reference_digests(golden, log_n):
    rec = next(r for r in golden["large"] if r["n"] == 1 << log_n)
    plan = nt.build_plan(rec["n"], bits=60, seed=0)
    assert plan.q == rec["q"]
    q, n = plan.q, plan.n
    a, b = rand(q, n, rec["a_seed"]), rand(q, n, rec["b_seed"])
    p = nt.Polynomial(a)
    nt.ntt_ct(p, plan)
    assert digest(p.numpy()) == rec["ntt_sha"]
    nt.intt_gs_scaled(p, plan)
    assert np.array_equal(p.numpy(), a)
    p = nt.Polynomial(a)
    nt.ntt_ct_truncated(p, plan)
    assert digest(p.numpy()) == rec["nttt_sha"]
    p = nt.Polynomial(rand(q, n, rec["intt_x_seed"]), "bit_reversed")
    nt.intt_gs(p, plan)
    assert digest(p.numpy()) == rec["intt_sha"]
    ctr = nt.OpCounter()
    c = nt.polymul_fused(dev(a), dev(b), nt.FusedPlan.from_plan(plan), ctr)
    assert digest(host(c)) == rec["fused_sha"]
    assert list(ctr.as_tuple()) == rec["fused_counts"]


@pytest.mark.parametrize("log_n", [2, 3, 5, 8, 9, 10, 11, 12, 13, 14, 16, 17])
@pytest.mark.parametrize("bits", [30, 62])
def test_fused_vs_oracle_many_sizes(log_n, bits):
    n = 1 << log_n
    plan = nt.build_plan(n, bits=bits, seed=3)
    B = 3
    A = np.stack([rand(plan.q, n, 100 + i) for i in range(B)])
    Bm = np.stack([rand(plan.q, n, 200 + i) for i in range(B)])
    tables = oracle.twiddles(plan.q, plan.psi, log_n)
    outs = nt.polymul_batch([(dev(A[i]), dev(Bm[i])) for i in range(B)], plan)
    for i in range(B):
        want = oracle.polymul_fused(A[i], Bm[i], plan.q, plan.psi, tables=tables)
        assert np.array_equal(host(outs[i]), want), (log_n, bits, i)


@pytest.mark.parametrize("log_n", [1, 2, 4, 9, 10, 11, 12, 13, 15, 17])
def test_transforms_batched_vs_oracle(log_n):
    n = 1 << log_n
    plan = nt.build_plan(n, bits=62, seed=5)
    red = plan.red_args
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    X = np.stack([rand(plan.q, n, 300 + i) for i in range(4)])
    t = dev(X)
    K.ntt_ct(t, plan.tw_fwd, *red, False)
    for i in range(4):
        w = X[i].copy()
        oracle.ntt_ct(w, f, *red, False)
        assert np.array_equal(host(t[i]), w), (log_n, i)
    for scaled in (False, True):
        t = dev(X)
        K.intt_gs(t, plan.tw_inv, plan.q, (plan.q + 1) // 2, *red[1:], scaled, False)
        for i in range(4):
            w = X[i].copy()
            oracle.intt_gs(w, v, plan.q, (plan.q + 1) // 2, *red[1:], scaled, False)
            assert np.array_equal(host(t[i]), w), (log_n, scaled, i)


def test_rns_batch_vs_oracle(golden):
    """cfg2 shape (N=2^14, 8 limbs) on a 4-ciphertext batch, every product."""
    g = next(b for b in golden["bases"] if b["n"] == 1 << 14)
    basis = nt.RnsBasis.build(g["n"], g["bits"], g["k"], seed=0)
    assert list(basis.primes) == g["primes"]
    assert [p.psi for p in basis.plans] == g["psis"]
    B, L, n = 4, g["k"], g["n"]
    A = np.stack([np.stack([rand(q, n, 10 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 999 + 10 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    got = host(nt.polymul_rns_batch(dev(A), dev(Bm), basis))
    want = oracle.polymul_rns(A, Bm, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)


def test_rns_cfg3_one_ciphertext(golden):
    """A full BASELINE cfg3 ciphertext: N=2^16, 21 x 60-bit limbs."""
    g = next(b for b in golden["bases"] if b["n"] == 1 << 16)
    basis = nt.RnsBasis.build(g["n"], 60, 21, seed=0)
    assert list(basis.primes) == g["primes"]
    n = g["n"]
    A = np.stack([rand(q, n, 7 + l) for l, q in enumerate(basis.primes)])[None]
    Bm = np.stack([rand(q, n, 70 + l) for l, q in enumerate(basis.primes)])[None]
    got = host(nt.polymul_rns_batch(dev(A), dev(Bm), basis))
    want = oracle.polymul_rns(A, Bm, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("log_n,limbs,batch", [(14, 8, 40), (16, 21, 7), (17, 32, 5)])
def test_split_stream_schedule(log_n, limbs, batch):
    """Large batches (>= 128 limb-products) run as two halves on internal
    streams with event fork/join (capi.cu run_polymul); the halves cut
    through a ciphertext when batch * limbs is odd.  The product equals the
    per-ciphertext (unsplit) calls and the oracle."""
    basis = nt.RnsBasis.build(1 << log_n, 60, limbs, seed=0)
    n = 1 << log_n
    A = np.stack([np.stack([rand(q, n, 13 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(batch)])
    Bm = np.stack([np.stack([rand(q, n, 4099 + 13 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(batch)])
    whole = host(nt.polymul_rns_batch(dev(A), dev(Bm), basis))
    each = np.stack([host(nt.polymul_rns_batch(dev(A[b:b + 1]), dev(Bm[b:b + 1]), basis))[0]
                     for b in range(batch)])
    assert np.array_equal(whole, each)
    k = 1 if log_n >= 16 else batch  # oracle on a subset at the large sizes
    want = oracle.polymul_rns(A[-k:], Bm[-k:], basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(whole[-k:], want)


def test_rns_host_buffers_streamed(golden):
    """Host (pinned and unpinned) [B, L, n] inputs stream through the
    chunked H2D / kernel / D2H pipeline: more chunks than device buffer sets,
    a ragged last chunk, results identical to the device-resident call."""
    g = next(b for b in golden["bases"] if b["n"] == 1 << 14)
    basis = nt.RnsBasis.build(g["n"], g["bits"], g["k"], seed=0)
    B, L, n = 7, g["k"], g["n"]
    A = np.stack([np.stack([rand(q, n, 31 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 577 + 31 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    want = host(nt.polymul_rns_batch(dev(A), dev(Bm), basis))
    assert np.array_equal(want[:2], oracle.polymul_rns(A[:2], Bm[:2], basis.primes,
                                                       [p.psi for p in basis.plans]))
    old = nt.rns.HOST_CHUNK_BYTES
    try:
        nt.rns.HOST_CHUNK_BYTES = 2 * L * n * 8  # 2 ciphertexts per chunk -> 4 chunks
        got = nt.polymul_rns_batch(torch.from_numpy(A).pin_memory(),
                                   torch.from_numpy(Bm).pin_memory(), basis)
        assert not got.is_cuda and np.array_equal(got.numpy(), want)
        got2 = nt.polymul_rns_batch(A, Bm, basis)  # numpy, unpinned
        assert np.array_equal(got2.numpy(), want)
    finally:
        nt.rns.HOST_CHUNK_BYTES = old
    empty = nt.polymul_rns_batch(A[:0], Bm[:0], basis)
    assert tuple(empty.shape) == (0, L, n)


def test_rns_bigint_end_to_end():
    basis = nt.RnsBasis.build(64, 30, 4, seed=2)
    import random

    rng = random.Random(11)
    for _ in range(3):
        a = [rng.randrange(basis.big_q) for _ in range(64)]
        b = [rng.randrange(basis.big_q) for _ in range(64)]
        assert nt.polymul_rns(a, b, basis) == nt.negacyclic_naive_bigint(a, b, basis.big_q)


def test_roundtrip_property_full_size():
    """ntt -> scaled intt is the identity on a large batch (size-independent)."""
    plan = nt.build_plan(1 << 17, bits=60, seed=0)
    X = torch.randint(0, 2**62, (6, 1 << 17), dtype=torch.int64, device="cuda")
    X = (X % plan.q).to(torch.uint64) if hasattr(torch, "uint64") else X
    orig = X.clone()
    K.ntt_ct(X, plan.tw_fwd, *plan.red_args, False)
    K.intt_gs(X, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:], True, False)
    assert torch.equal(X.cpu(), orig.cpu())


def test_edge_cases():
    plan = nt.build_plan(4096, bits=60, seed=0)
    empty = torch.empty((0, 4096), dtype=torch.uint64, device="cuda")
    K.ntt_ct(empty, plan.tw_fwd, *plan.red_args, False)  # empty batch: no-op
    with pytest.raises(ValueError):
        K.ntt_ct(torch.zeros(1000, dtype=torch.uint64, device="cuda"), plan.tw_fwd,
                 *plan.red_args, False)
    with pytest.raises(ValueError):
        nt.polymul_fused([0] * 8, [0] * 4096, plan)
    # wraparound sign: x^(n-1) * x = -1
    p8 = nt.build_plan(8, bits=12, seed=0)
    a = [0] * 8
    b = [0] * 8
    a[7] = 1
    b[1] = 1
    assert nt.polymul_fused(a, b, p8).tolist() == [p8.q - 1] + [0] * 7
    # unit impulse -> flat spectrum
    p32 = nt.build_plan(32, bits=14, seed=0)
    u = nt.Polynomial.unit(32)
    nt.ntt_ct(u, p32)
    assert u.to_list() == [1] * 32
    # ordering discipline
    with pytest.raises(ValueError):
        nt.ntt_ct(u, p32)


def test_mulmod_loop_and_tensor_mulmod(golden):
    for s in golden["mulmod_loop"]:
        q = s["q"]
        a, b = rand(q, s["n"], s["a_seed"]), rand(q, s["n"], s["b_seed"])
        mod = nt.Modulus(q)
        red = mod.reduction_params(s["variant"])
        assert K.mulmod_loop(dev(a), dev(b), q, *red, s["passes"]) == s["sink"]
        prod = nt.mulmod(dev(a), dev(b), mod, s["variant"])
        assert np.array_equal(host(prod), (a.astype(object) * b.astype(object) % q)
                              .astype(np.uint64))


def test_batch_ntt_deterministic_any_workers():
    plan = nt.build_plan(128, bits=30, seed=0)
    import random

    rng = random.Random(42)
    rows = [nt.Polynomial.random(plan, rng) for _ in range(24)]
    base = [r.numpy() for r in nt.batch_ntt([r.copy() for r in rows], plan, 1)]
    for w in (2, 8):
        out = nt.batch_ntt([r.copy() for r in rows], plan, w)
        assert all(np.array_equal(x, y.numpy()) for x, y in zip(base, out))


@pytest.mark.parametrize("bits", [24, 30, 59, 60, 61, 62])
@pytest.mark.parametrize("log_n", [10, 13, 16])
def test_lazy_bound_paths_vs_oracle(bits, log_n):
    """Every lazy-reduction regime: [0,16q) forward (q < 2^60), [0,8q)
    (q < 2^61) and Harvey [0,4q) (62-bit) through the fused RNS path and the
    standalone transforms."""
    n = 1 << log_n
    basis = nt.RnsBasis.build(n, bits, 2, seed=4)
    B = 2
    A = np.stack([np.stack([rand(q, n, 5 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 50 + 5 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    # adversarial extremes: all q-1
    A[0, 0, :] = basis.primes[0] - 1
    Bm[0, 0, :] = basis.primes[0] - 1
    got = host(nt.polymul_rns_batch(dev(A), dev(Bm), basis))
    want = oracle.polymul_rns(A, Bm, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)
    plan = basis.plans[1]
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    x = A[1, 1].copy()
    t = dev(x)
    K.ntt_ct(t, plan.tw_fwd, *plan.red_args, False)
    w = x.copy()
    oracle.ntt_ct(w, f, *plan.red_args, False)
    assert np.array_equal(host(t), w)
    K.intt_gs(t, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:], True, False)
    assert np.array_equal(host(t), x)


# ---- verification kernels and alternative transform shapes ----------------

def test_negacyclic_naive_matches_reference(golden, vectors):
    for c in golden["vector_cases"]:
        key = c["key"]
        a, b = vectors[key + "_a"], vectors[key + "_b"]
        ctr = nt.OpCounter()
        got = nt.negacyclic_naive(dev(a), dev(b), c["q"], ctr)
        assert np.array_equal(host(got), vectors[key + "_naive"]), key
        assert list(ctr.as_tuple()) == c["naive_counts"], key
        # host arrays in -> host array out, like the reference
        assert np.array_equal(nt.negacyclic_naive(a, b, c["q"]), vectors[key + "_naive"])
        # the fused product equals the schoolbook oracle
        assert np.array_equal(vectors[key + "_fused"], vectors[key + "_naive"]), key


def test_negacyclic_naive_batch_and_wraparound():
    q = 998244353
    n = 64
    a = np.zeros((3, n), dtype=np.uint64)
    b = np.zeros((3, n), dtype=np.uint64)
    a[:, n - 1] = 1
    b[:, 1] = 1  # x^(n-1) * x = -1
    got = host(nt.negacyclic_naive(dev(a), dev(b), q))
    want = np.zeros((3, n), dtype=np.uint64)
    want[:, 0] = q - 1
    assert np.array_equal(got, want)


def test_radix4_and_2d_shapes_match_reference(golden, vectors):
    for c in golden["vector_cases"]:
        key, n = c["key"], c["n"]
        plan = _plan(c)
        a, x = vectors[key + "_a"], vectors[key + "_x"]
        if "r4_counts" in c:
            ctr = nt.OpCounter()
            p = nt.ntt_radix4(nt.Polynomial(a.copy()), plan, ctr)
            assert np.array_equal(p.numpy(), vectors[key + "_r4"]), key
            assert list(ctr.as_tuple()) == c["r4_counts"], key
            ctr = nt.OpCounter()
            p = nt.intt_radix4(nt.Polynomial(x.copy(), "bit_reversed"), plan, ctr)
            assert np.array_equal(p.numpy(), vectors[key + "_ir4"]), key
            assert list(ctr.as_tuple()) == c["ir4_counts"], key
        else:
            with pytest.raises(ValueError):
                nt.ntt_radix4(nt.Polynomial(a.copy()), plan)
        ctr = nt.OpCounter()
        p = nt.ntt_2d(nt.Polynomial(a.copy()), plan, ctr)
        assert p.ordering == "vendor_2d"
        assert np.array_equal(p.numpy(), vectors[key + "_2d"]), key
        assert list(ctr.as_tuple()) == c["2d_counts"], key
        ctr = nt.OpCounter()
        p = nt.ntt_2d_inv(nt.Polynomial(x.copy(), "vendor_2d"), plan, ctr)
        assert np.array_equal(p.numpy(), vectors[key + "_2di"]), key
        assert list(ctr.as_tuple()) == c["2di_counts"], key
        # round trip and the documented permutation identity
        p = nt.ntt_2d_inv(nt.ntt_2d(nt.Polynomial(a.copy()), plan), plan)
        assert np.array_equal(p.numpy(), a), key
        perm = nt.ntt_2d_permutation(plan)
        assert np.array_equal(vectors[key + "_2d"], vectors[key + "_ntt"][perm]), key


def test_2d_full_size_roundtrip():
    plan = nt.build_plan(1 << 16, bits=60, seed=0)
    a = rand(plan.q, 1 << 16, 5)
    p = nt.ntt_2d(nt.Polynomial(a.copy()), plan)
    ref = nt.ntt_ct(nt.Polynomial(a.copy()), plan).numpy()
    assert np.array_equal(p.numpy(), ref[nt.ntt_2d_permutation(plan)])
    assert np.array_equal(nt.ntt_2d_inv(p, plan).numpy(), a)


def test_sweeps_match_reference(golden):
    for s in golden["sweeps"]:
        t = np.zeros((3, 4), dtype=np.uint64)
        if s["kind"] == "exhaustive":
            mism, first = K.sweep_exhaustive(s["q_lo"], s["q_hi"], t)
        else:
            mism, first = K.sweep_random(s["bits"], s["samples"], s["seed"], t)
        assert mism == s["mism"], s
        assert (list(first) if first else None) == s["first"], s
        assert [[int(v) for v in r] for r in t] == s["tallies"], s
        # tallies accumulate like the reference
        if s["kind"] == "random" and s["bits"] == 30:
            K.sweep_random(s["bits"], s["samples"], s["seed"], t)
            assert [[int(v) for v in r] for r in t] == [[2 * v for v in r] for r in s["tallies"]]


# ---- RNS decomposition / CRT reconstruction on the GPU --------------------

def _big_values(big_q, n, seed):
    import random

    rng = random.Random(seed)
    vals = [rng.randrange(big_q) for _ in range(n)]
    vals[:4] = [0, 1, big_q - 1, big_q // 2]  # edges
    return vals


@pytest.mark.parametrize("n,bits,limbs", [(64, 30, 4), (4096, 60, 21), (1024, 60, 32),
                                          (256, 62, 3), (128, 20, 7)])
def test_crt_decompose_reconstruct_match_oracle(n, bits, limbs):
    basis = nt.RnsBasis.build(max(n, 4), bits, limbs, seed=1)
    vals = _big_values(basis.big_q, n, n + limbs)
    want = oracle.crt_decompose(vals, basis.primes)
    got = np.stack(nt.decompose(vals, basis))
    assert np.array_equal(got, want)
    # reconstruct arbitrary canonical residues (not just round trips)
    rng = np.random.default_rng(n)
    res = np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in basis.primes])
    assert nt.reconstruct(list(res), basis) == oracle.crt_reconstruct(res, basis.primes)
    assert nt.reconstruct(list(got), basis) == vals


def test_polymul_rns_bigint_vs_schoolbook():
    basis = nt.RnsBasis.build(256, 60, 21, seed=0)
    a = _big_values(basis.big_q, 256, 1)
    b = _big_values(basis.big_q, 256, 2)
    assert nt.polymul_rns(a, b, basis) == nt.negacyclic_naive_bigint(a, b, basis.big_q)


def test_polymul_rns_words_cfg3_residue_consistency(golden):
    """Full cfg3 size (N=2^16, 21 limbs, 2 ciphertexts of big integers):
    decompose(result) equals the oracle's per-limb products of the decomposed
    inputs (a size-independent check of decompose + polymul + CRT)."""
    basis = nt.RnsBasis.build(1 << 16, 60, 21, seed=0)
    W = nt.rns.num_words(basis)
    rng = np.random.default_rng(3)
    Aw = rng.integers(0, 2**63, (2, 1 << 16, W), dtype=np.uint64)
    Bw = rng.integers(0, 2**63, (2, 1 << 16, W), dtype=np.uint64)
    top = nt.ints_to_words([basis.big_q - 1], W)[0]
    Aw[:, :, -1] %= top[-1]  # keep every coefficient below big_q
    Bw[:, :, -1] %= top[-1]
    Cw = nt.polymul_rns_words(dev(Aw), dev(Bw), basis)
    ra = host(nt.crt_decompose(dev(Aw), basis))
    rb = host(nt.crt_decompose(dev(Bw), basis))
    rc = host(nt.crt_decompose(Cw, basis))
    want = oracle.polymul_rns(ra[:1], rb[:1], basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(rc[:1], want)
    # every output coefficient is the canonical representative (< big_q)
    assert max(nt.words_to_ints(host(Cw[1])[:512])) < basis.big_q


# ---- verification suites (reference verify.py / test_acceptance.py) -------

def test_acceptance_reduction_criteria():
    """Criteria 1-4 of the reference acceptance gate on the GPU sweeps:
    exhaustive q in [3, 255], 10^6 random samples per bit size, subtraction
    bounds, classical second-subtraction frequency."""
    V = nt.verify
    t = np.zeros((3, 4), dtype=np.uint64)
    r = V.reduction_exhaustive(3, 255, t)
    assert r.passed, r.line()
    for bits in (28, 29, 30, 62):
        t = np.zeros((3, 4), dtype=np.uint64)
        r = V.reduction_random(bits, 1_000_000, 42, t)
        assert r.passed, r.line()
        if bits == 30:
            frac = r.measurements["classical_two_sub_fraction"]
            assert 0 < frac < 0.05
    # a failing configuration is reported with the reference's message shape
    r = V.reduction_random(63, 1000, 6)
    assert not r.passed and "mismatches; first: proposed(" in r.detail


def test_verify_suites_pass():
    res = nt.verify.run_all(samples=1000)
    assert [x.status for x in res] == ["PASS"] * len(res), [x.line() for x in res]
    names = [x.name for x in res]
    assert names[0] == "reduction-exhaustive q in [3, 255]"
    assert "polymul-three-way x100" in names and "rns-roundtrip x20" in names


@pytest.mark.parametrize("log_n,limbs,batch", [(14, 8, 64), (16, 21, 64), (17, 32, 8)])
def test_baseline_configs_full_batch(log_n, limbs, batch):
    """BASELINE cfg2 (N=2^14, 8 limbs, 64 products), cfg3 at bench.py's
    default batch (N=2^16, 21 limbs, 64 ciphertexts = the two-stream split)
    and cfg4 (N=2^17, 32 limbs, 8 ciphertexts) at full size: first and last ciphertext against the
    oracle, and bilinearity c(a, b1 + b2) = c(a, b1) + c(a, b2) mod q over the
    whole batch (a size-independent check of every product)."""
    basis = nt.RnsBasis.build(1 << log_n, 60, limbs, seed=0)
    n = 1 << log_n
    q = torch.tensor(np.array(basis.primes, dtype=np.uint64).astype(np.int64),
                     device="cuda").view(1, limbs, 1)
    g = torch.Generator(device="cuda").manual_seed(log_n)

    def rnd():
        x = torch.randint(0, 2**62, (batch, limbs, n), dtype=torch.int64, device="cuda",
                          generator=g)
        return (x % q).to(torch.uint64)

    A, B1, B2 = rnd(), rnd(), rnd()
    B12 = ((B1.to(torch.int64) + B2.to(torch.int64)) % q).to(torch.uint64)
    C1 = nt.polymul_rns_batch(A, B1, basis)
    C2 = nt.polymul_rns_batch(A, B2, basis)
    C12 = nt.polymul_rns_batch(A, B12, basis)
    # (C1 + C2) mod q, in int64 without overflow (values < 2^60)
    S = ((C1.to(torch.int64) + C2.to(torch.int64)) % q).to(torch.uint64)
    assert torch.equal(S, C12)
    psis = [p.psi for p in basis.plans]
    for i in (0, batch - 1):
        want = oracle.polymul_rns(host(A[i:i + 1]), host(B1[i:i + 1]), basis.primes, psis)
        assert np.array_equal(host(C1[i:i + 1]), want), i
