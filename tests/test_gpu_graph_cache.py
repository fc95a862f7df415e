"""GPU checks of the launch-graph cache (csrc/capi.cu run_graphed): a call
repeated with identical arguments is replayed from a captured CUDA graph from
its second occurrence on.  The replay must read the buffers' CURRENT
contents, follow schedule-knob changes, order correctly with other work on
the caller's stream, and stay out of the way while the caller itself is
capturing a graph.  Every result is compared with the C oracle."""

from __future__ import annotations

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


def _fwd_ref(rows, plan, truncate=False):
    f, _ = oracle.twiddles(plan.q, plan.psi, plan.log_n)
    want = rows.copy()
    for w in want:
        oracle.ntt_ct(w, f, *plan.red_args, truncate)
    return want


@pytest.mark.parametrize("log_n", [13, 16, 17])
def test_replay_reads_current_contents(log_n):
    """Same pointers, new data every call: each result is the transform of
    that call's data (the graph binds addresses, not values)."""
    n = 1 << log_n
    plan = nt.build_plan(n, bits=60, seed=3)
    x = torch.empty((1, n), dtype=torch.uint64, device="cuda")
    for i in range(5):
        rows = rand(plan.q, n, 50 + i)[None]
        x.copy_(torch.from_numpy(rows))
        nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
        assert np.array_equal(x.cpu().numpy(), _fwd_ref(rows, plan)), f"call {i}"
        nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:], True,
                           False, None)
        assert np.array_equal(x.cpu().numpy(), rows), f"round trip {i}"


def test_replay_follows_schedule_changes():
    """A schedule change between two identical calls is honoured (the knob
    invalidates captured graphs); every schedule gives the same answer."""
    n = 1 << 15
    plan = nt.build_plan(n, bits=59, seed=5)
    rows = rand(plan.q, n, 7)[None]
    want = _fwd_ref(rows, plan)
    x = torch.empty((1, n), dtype=torch.uint64, device="cuda")
    try:
        for sched in (lib.SCHED_AUTO, lib.SCHED_THREE, lib.SCHED_PASSES, lib.SCHED_CLUSTER,
                      lib.SCHED_AUTO):
            lib.call("nttmul_set_schedule", 1, 15, sched)
            for _ in range(3):
                x.copy_(torch.from_numpy(rows))
                nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
                assert np.array_equal(x.cpu().numpy(), want), f"schedule {sched}"
    finally:
        lib.call("nttmul_set_schedule", 1, 15, lib.SCHED_AUTO)


def test_replay_orders_with_stream_work():
    """Back-to-back replays on a side stream, interleaved with torch copies
    on that stream and no host synchronisation in between: a chain of
    forward / inverse pairs returns the input."""
    n = 1 << 14
    plan = nt.build_plan(n, bits=60, seed=8)
    rows = np.stack([rand(plan.q, n, 90 + i) for i in range(2)])
    src = torch.from_numpy(rows).cuda()
    x = torch.empty_like(src)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(20):
            x.copy_(src)
            nt.kernels.ntt_ct(x, plan.tw_fwd, *plan.red_args, False, None)
            nt.kernels.intt_gs(x, plan.tw_inv, plan.q, (plan.q + 1) // 2, *plan.red_args[1:],
                               True, False, None)
            src.copy_(x)
    s.synchronize()
    assert np.array_equal(src.cpu().numpy(), rows)


def test_fused_product_replays_and_user_capture():
    """The fused RNS product through repeated identical calls, and inside a
    torch.cuda.CUDAGraph capture by the caller (the library launches
    directly into the caller's capture)."""
    n = 1 << 14
    basis = nt.RnsBasis.build(n, 60, 3, seed=0)
    A = np.stack([rand(q, n, 3 + l) for l, q in enumerate(basis.primes)])[None]
    B = np.stack([rand(q, n, 300 + l) for l, q in enumerate(basis.primes)])[None]
    want = oracle.polymul_rns(A, B, basis.primes, [p.psi for p in basis.plans])
    da, db = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty_like(da)
    for _ in range(4):
        out.zero_()
        nt.polymul_rns_batch(da, db, basis, out=out)
        assert np.array_equal(out.cpu().numpy(), want)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        nt.polymul_rns_batch(da, db, basis, out=out)  # warm the wrapper's caches
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        nt.polymul_rns_batch(da, db, basis, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)


def test_grid_launches_on_concurrent_streams():
    """One-launch grid transforms and fused products issued from four
    streams at once (each its own buffers, no host synchronisation), plus a
    caller-captured CUDA graph of grid launches replayed concurrently: every
    launch picks its own barrier word (csrc/grid_kernels.cuh launch_slot),
    so all round trips come back exact."""
    n = 1 << 15
    plan = nt.build_plan(n, bits=60, seed=12)
    fused = nt.FusedPlan.from_plan(plan)
    inv_args = (plan.q, (plan.q + 1) // 2, *plan.red_args[1:], True, False, None)
    bufs = [torch.from_numpy(rand(plan.q, n, 700 + i)[None]).cuda() for i in range(5)]
    refs = [b.clone() for b in bufs]
    prod_a = torch.from_numpy(rand(plan.q, n, 800)).cuda()
    prod_b = torch.from_numpy(rand(plan.q, n, 801)).cuda()
    want_prod = oracle.polymul_rns(rand(plan.q, n, 800)[None, None], rand(plan.q, n, 801)[None, None],
                                   [plan.q], [plan.psi])[0, 0]
    # a captured graph of forward + inverse on buffer 4
    gstream = torch.cuda.Stream()
    gstream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(gstream):
        nt.kernels.ntt_ct(bufs[4], plan.tw_fwd, *plan.red_args, False, None)
        nt.kernels.intt_gs(bufs[4], plan.tw_inv, *inv_args)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gstream):
        nt.kernels.ntt_ct(bufs[4], plan.tw_fwd, *plan.red_args, False, None)
        nt.kernels.intt_gs(bufs[4], plan.tw_inv, *inv_args)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    prods = []
    for it in range(25):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                nt.kernels.ntt_ct(bufs[i], plan.tw_fwd, *plan.red_args, False, None)
                nt.kernels.intt_gs(bufs[i], plan.tw_inv, *inv_args)
                if i == 0 and it % 5 == 0:
                    prods.append(nt.polymul_fused(prod_a, prod_b, fused))
        with torch.cuda.stream(gstream):
            g.replay()
    torch.cuda.synchronize()
    for i in range(5):
        assert np.array_equal(bufs[i].cpu().numpy(), refs[i].cpu().numpy()), f"buffer {i}"
    for p in prods:
        assert np.array_equal(p.cpu().numpy(), want_prod)
