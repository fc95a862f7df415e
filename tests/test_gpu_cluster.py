"""GPU parity of the thread-block-cluster schedule (csrc/cluster_kernels.cuh):
one cluster of n / 4096 CTAs per polynomial, rows in distributed shared
memory.  Forced on with nttmul_set_schedule and compared bit-for-bit with
the C oracle and with the three-launch column / row / column schedule, for
the fused product (n = 2^13 .. 2^16, ragged batches, every cluster size) and
the standalone transforms (ntt_ct full / truncated, intt_gs scaled / plain /
skip_first)."""

from __future__ import annotations

import contextlib

import numpy as np
import pytest
import torch

import oracle
from conftest import rand

pytestmark = pytest.mark.gpu

nt = pytest.importorskip("paper_2209_01290_b200")
lib = nt._lib


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64)).cuda()


@contextlib.contextmanager
def schedule(which, log_n, sched):
    lib.call("nttmul_set_schedule", which, log_n, sched)
    try:
        yield
    finally:
        lib.call("nttmul_set_schedule", which, log_n, lib.SCHED_AUTO)


@pytest.mark.parametrize("log_n,L,B", [(13, 3, 3), (14, 8, 5), (15, 2, 3), (16, 21, 1),
                                       (16, 3, 6)])
def test_cluster_fused_product(log_n, L, B):
    n = 1 << log_n
    basis = nt.RnsBasis.build(n, 60, L, seed=0)
    A = np.stack([np.stack([rand(q, n, 11 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 909 + 11 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    with schedule(0, log_n, lib.SCHED_CLUSTER):
        got = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    with schedule(0, log_n, lib.SCHED_THREE):
        three = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    assert np.array_equal(got, three)
    k = min(B, 2)
    want = oracle.polymul_rns(A[:k], Bm[:k], basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got[:k], want)


def test_cluster_fused_edge_values():
    """q - 1 everywhere and x^(n-1) * x = -1 through the cluster path."""
    n = 1 << 14
    basis = nt.RnsBasis.build(n, 60, 2, seed=0)
    q = np.array(basis.primes, dtype=np.uint64)[None, :, None]
    A = np.broadcast_to(q - 1, (1, 2, n)).copy()
    X = np.zeros((1, 2, n), dtype=np.uint64)
    Y = np.zeros((1, 2, n), dtype=np.uint64)
    X[..., n - 1] = 1
    Y[..., 1] = 1
    with schedule(0, 14, lib.SCHED_CLUSTER):
        got = nt.polymul_rns_batch(dev(A), dev(A), basis).cpu().numpy()
        wrap = nt.polymul_rns_batch(dev(X), dev(Y), basis).cpu().numpy()
    want = oracle.polymul_rns(A, A, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)
    assert np.array_equal(wrap[..., 0], (q - 1)[..., 0]) and not wrap[..., 1:].any()


@pytest.mark.parametrize("log_n", [13, 14, 15, 16])
def test_cluster_standalone_transforms(log_n):
    n = 1 << log_n
    plan = nt.build_plan(n, bits=59, seed=1)
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    rows = np.stack([rand(plan.q, n, 7 + i) for i in range(3)])
    args = plan.red_args
    for truncate in (False, True):
        want = rows.copy()
        for w in want:
            oracle.ntt_ct(w, f, *args, truncate)
        x = dev(rows)
        with schedule(1, log_n, lib.SCHED_CLUSTER):
            nt.kernels.ntt_ct(x, plan.tw_fwd, *args, truncate, None)
        assert np.array_equal(x.cpu().numpy(), want), f"ntt_ct truncate={truncate}"
    half_q = (plan.q + 1) // 2
    for scaled, skip in ((True, False), (False, False), (True, True)):
        want = rows.copy()
        for w in want:
            oracle.intt_gs(w, v, plan.q, half_q, *args[1:], scaled, skip)
        x = dev(rows)
        with schedule(1, log_n, lib.SCHED_CLUSTER):
            nt.kernels.intt_gs(x, plan.tw_inv, plan.q, half_q, *args[1:], scaled, skip, None)
        assert np.array_equal(x.cpu().numpy(), want), f"intt_gs scaled={scaled} skip={skip}"


def test_schedule_knob_rejects_bad_arguments():
    for args in ((2, 14, 1), (0, 12, 1), (0, 17, 2), (0, 14, 3), (0, 14, 5), (1, 14, 5),
                 (1, 18, 1), (1, 17, 2)):
        with pytest.raises(nt._lib.NttmulError):
            lib.call("nttmul_set_schedule", *args)


# ---- radix splits (nttmul_set_split, BASELINE cfg5) ------------------------

@contextlib.contextmanager
def split(log_n, log_r):
    lib.call("nttmul_set_split", log_n, log_r)
    try:
        yield
    finally:
        lib.call("nttmul_set_split", log_n, 0)


@pytest.mark.parametrize("log_n,log_r", [(13, 10), (13, 11), (14, 10), (14, 13), (15, 11),
                                         (15, 13), (16, 11), (16, 13), (17, 13)])
def test_radix_splits_bit_exact(log_n, log_r):
    n = 1 << log_n
    basis = nt.RnsBasis.build(n, 60, 2, seed=0)
    A = np.stack([np.stack([rand(q, n, 5 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(2)])
    Bm = np.stack([np.stack([rand(q, n, 77 + 5 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(2)])
    with split(log_n, log_r), schedule(0, log_n, lib.SCHED_THREE) if log_n <= 16 else \
            contextlib.nullcontext():
        got = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    want = oracle.polymul_rns(A[:1], Bm[:1], basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got[:1], want)
    plan = basis.plans[0]
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    rows = A[:, 0].copy()
    want = rows.copy()
    for w in want:
        oracle.ntt_ct(w, f, *plan.red_args, False)
    x = dev(rows)
    with split(log_n, log_r), schedule(1, log_n, lib.SCHED_THREE) if log_n <= 16 else \
            contextlib.nullcontext():
        nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
        assert np.array_equal(x.cpu().numpy(), want)
        nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:],
                           True, False, None)
    assert np.array_equal(x.cpu().numpy(), rows)


def test_split_knob_rejects_bad_arguments():
    for args in ((12, 10), (14, 9), (14, 14), (17, 11), (18, 13)):
        with pytest.raises(nt._lib.NttmulError):
            lib.call("nttmul_set_split", *args)


@pytest.mark.parametrize("log_n", [13, 14, 15, 16, 17])
@pytest.mark.parametrize("batch", [1, 3])
def test_latency_pass_schedule_bit_exact(log_n, batch):
    """Strided column passes of <= 3 stages + 1024-word rows
    (NTTMUL_SCHED_PASSES) for ntt_ct (full / truncated) and intt_gs (scaled
    full / skip_first / plain)."""
    n = 1 << log_n
    plan = nt.build_plan(n, bits=60, seed=2)
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    rows = np.stack([rand(plan.q, n, 31 + i) for i in range(batch)])
    args = plan.red_args
    half_q = (plan.q + 1) // 2
    with schedule(1, log_n, lib.SCHED_PASSES):
        for truncate in (False, True):
            want = rows.copy()
            for w in want:
                oracle.ntt_ct(w, f, *args, truncate)
            x = dev(rows)
            nt.kernels.ntt_ct(x, plan.tw_fwd, *args, truncate, None)
            assert np.array_equal(x.cpu().numpy(), want), f"ntt_ct truncate={truncate}"
        for scaled, skip in ((True, False), (True, True), (False, False)):
            want = rows.copy()
            for w in want:
                oracle.intt_gs(w, v, plan.q, half_q, *args[1:], scaled, skip)
            x = dev(rows)
            nt.kernels.intt_gs(x, plan.tw_inv, plan.q, half_q, *args[1:], scaled, skip, None)
            assert np.array_equal(x.cpu().numpy(), want), f"intt scaled={scaled} skip={skip}"


@pytest.mark.parametrize("log_n,batch", [(13, 131), (16, 128)])
def test_batched_transforms_large_batches(log_n, batch):
    """Large batches of standalone transforms (odd counts, > one wave of
    row CTAs): every row equals the oracle's transform and round-trips."""
    n = 1 << log_n
    plan = nt.build_plan(n, bits=60, seed=4)
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    base = np.stack([rand(plan.q, n, 900 + i) for i in range(3)])
    rows = base[np.arange(batch) % 3]
    want = base.copy()
    for w in want:
        oracle.ntt_ct(w, f, *plan.red_args, False)
    x = dev(rows)
    nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
    got = x.cpu().numpy()
    assert np.array_equal(got, want[np.arange(batch) % 3])
    nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:], True,
                       False, None)
    assert np.array_equal(x.cpu().numpy(), rows)


# ---- one-launch grid schedule (NTTMUL_SCHED_GRID, csrc/grid_kernels.cuh) ---

@pytest.mark.parametrize("bits", [59, 61, 62])  # lazy bounds 16, 8, 4
@pytest.mark.parametrize("log_n", [13, 14, 15, 16, 17])
@pytest.mark.parametrize("batch", [1, 3])
def test_grid_schedule_bit_exact(log_n, batch, bits):
    """The cooperative one-launch transform for ntt_ct (full / truncated)
    and intt_gs (scaled full / skip_first / plain), every lazy-bound class
    of moduli, single and batched (ragged) launches."""
    n = 1 << log_n
    plan = nt.build_plan(n, bits=bits, seed=3)
    f, v = oracle.twiddles(plan.q, plan.psi, log_n)
    rows = np.stack([rand(plan.q, n, 61 + i) for i in range(batch)])
    args = plan.red_args
    half_q = (plan.q + 1) // 2
    with schedule(1, log_n, lib.SCHED_GRID):
        for truncate in (False, True):
            want = rows.copy()
            for w in want:
                oracle.ntt_ct(w, f, *args, truncate)
            x = dev(rows)
            nt.kernels.ntt_ct(x, plan.tw_fwd, *args, truncate, None)
            assert np.array_equal(x.cpu().numpy(), want), f"ntt_ct truncate={truncate}"
        for scaled, skip in ((True, False), (True, True), (False, False)):
            want = rows.copy()
            for w in want:
                oracle.intt_gs(w, v, plan.q, half_q, *args[1:], scaled, skip)
            x = dev(rows)
            nt.kernels.intt_gs(x, plan.tw_inv, plan.q, half_q, *args[1:], scaled, skip, None)
            assert np.array_equal(x.cpu().numpy(), want), f"intt scaled={scaled} skip={skip}"


def test_grid_schedule_edge_values():
    """All-(q-1) input and a lone x^(n-1) through the grid transforms: the
    forward / inverse round trip returns them and the forward matches the
    oracle (largest lazy intermediates)."""
    n = 1 << 16
    plan = nt.build_plan(n, bits=59, seed=9)
    f, _ = oracle.twiddles(plan.q, plan.psi, 16)
    top = np.full((1, n), plan.q - 1, dtype=np.uint64)
    mono = np.zeros((1, n), dtype=np.uint64)
    mono[0, n - 1] = 1
    with schedule(1, 16, lib.SCHED_GRID):
        for rows in (top, mono):
            want = rows.copy()
            oracle.ntt_ct(want[0], f, *plan.red_args, False)
            x = dev(rows)
            nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
            assert np.array_equal(x.cpu().numpy(), want)
            nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:],
                               True, False, None)
            assert np.array_equal(x.cpu().numpy(), rows)


def test_grid_schedule_rejects_oversized_batch():
    """A forced grid launch larger than the co-resident CTA count fails
    loudly (no silent deadlock, no fallback)."""
    n = 1 << 17
    plan = nt.build_plan(n, bits=59, seed=1)
    x = torch.zeros((64, n), dtype=torch.uint64, device="cuda")
    with schedule(1, 17, lib.SCHED_GRID):
        with pytest.raises(nt._lib.NttmulError):
            nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)


@pytest.mark.parametrize("variant", ["proposed", "classical", "builtin"])
@pytest.mark.parametrize("bits", [40, 59, 61, 62])
@pytest.mark.parametrize("log_n", [13, 14, 15, 16, 17])
def test_grid_fused_product_bit_exact(log_n, bits, variant):
    """The one-launch fused product (forward columns, rows + Karatsuba
    middle, inverse columns) for every reduction variant and lazy-bound
    class, forced on and in auto (up to 4 limb-products), against the
    three-launch schedule and the oracle."""
    n = 1 << log_n
    # a forced grid launch must fit co-resident: 2 limb-products (one at
    # 2^17, whose 512-thread CTAs run one per SM)
    L, B = (1, 1) if log_n == 17 else (2, 1)
    basis = nt.RnsBasis.build(n, bits, L, seed=1, variant=variant)
    A = np.stack([np.stack([rand(q, n, 17 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 404 + 17 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    with schedule(0, log_n, lib.SCHED_THREE):
        three = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    with schedule(0, log_n, lib.SCHED_GRID):
        got = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    auto = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    assert np.array_equal(got, three) and np.array_equal(auto, three)
    want = oracle.polymul_rns(A, Bm, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)


def test_grid_fused_edge_values_and_aliasing():
    """q - 1 everywhere, x^(n-1) * x = -1, and c aliasing a, through the
    forced one-launch fused product."""
    n = 1 << 16
    basis = nt.RnsBasis.build(n, 60, 2, seed=0)
    q = np.array(basis.primes, dtype=np.uint64)[None, :, None]
    top = np.broadcast_to(q - 1, (1, 2, n)).copy()
    X = np.zeros((1, 2, n), dtype=np.uint64)
    Y = np.zeros((1, 2, n), dtype=np.uint64)
    X[..., n - 1] = 1
    Y[..., 1] = 1
    with schedule(0, 16, lib.SCHED_GRID):
        got = nt.polymul_rns_batch(dev(top), dev(top), basis).cpu().numpy()
        wrap = nt.polymul_rns_batch(dev(X), dev(Y), basis).cpu().numpy()
        da = dev(X)
        nt.polymul_rns_batch(da, dev(Y), basis, out=da)
        inplace = da.cpu().numpy()
    want = oracle.polymul_rns(top, top, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)
    assert np.array_equal(wrap[..., 0], (q - 1)[..., 0]) and not wrap[..., 1:].any()
    assert np.array_equal(inplace, wrap)


@pytest.mark.parametrize("log_n,L,B", [(13, 8, 4), (14, 4, 2), (15, 8, 1)])
def test_grid_fused_auto_larger_counts(log_n, L, B):
    """Auto picks the one-launch fused product up to its per-size limit
    (2^13: 32 limb-products, 2^14 / 2^15: 8): same result as three launches
    and as the oracle."""
    n = 1 << log_n
    basis = nt.RnsBasis.build(n, 60, L, seed=2)
    A = np.stack([np.stack([rand(q, n, 5 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 55 + 5 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    auto = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    with schedule(0, log_n, lib.SCHED_THREE):
        three = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    assert np.array_equal(auto, three)
    want = oracle.polymul_rns(A[:1], Bm[:1], basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(auto[:1], want)
