"""GPU: API hardening of the drop-in surface - caller-supplied buffers are
validated before any launch, the twiddle-pair cache is bounded and never
keeps a table alive, mixed-variant bases (accepted by the reference,
rns.py:61-73) multiply bit-exactly, device caches follow the current
device."""

from __future__ import annotations

import gc

import numpy as np
import pytest
import torch

import oracle
from conftest import rand

pytestmark = pytest.mark.gpu

nt = pytest.importorskip("paper_2209_01290_b200")
K = nt.kernels


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64)).cuda()


def _batch(basis, B, seed):
    n = basis.n
    return np.stack([np.stack([rand(q, n, seed + 31 * b + l) for l, q in enumerate(basis.primes)])
                     for b in range(B)])


@pytest.mark.parametrize("log_n", [12, 14])
def test_out_and_workspace_are_validated(log_n):
    basis = nt.RnsBasis.build(1 << log_n, 60, 2, seed=0)
    A, Bm = dev(_batch(basis, 2, 1)), dev(_batch(basis, 2, 99))
    want = nt.polymul_rns_batch(A, Bm, basis)
    bad = [
        torch.empty(A.shape, dtype=torch.int64, device="cuda"),           # dtype
        torch.empty((2, 2, (1 << log_n) // 2), dtype=torch.uint64, device="cuda"),  # shape
        torch.empty((2, 2, 2 << log_n), dtype=torch.uint64, device="cuda")[..., ::2],  # strided
        torch.empty(A.shape, dtype=torch.uint64),                         # host
    ]
    for t in bad:
        with pytest.raises(ValueError):
            nt.polymul_rns_batch(A, Bm, basis, out=t)
        with pytest.raises(ValueError):
            nt.polymul_rns_batch(A, Bm, basis, workspace=t)
    with pytest.raises(ValueError):
        nt.polymul_rns_batch(A, Bm, basis, workspace=A)
    out, ws = torch.empty_like(A), torch.empty_like(A)
    got = nt.polymul_rns_batch(A, Bm, basis, out=out, workspace=ws)
    assert got is out and torch.equal(out, want)
    # host path: a 4-byte dtype `out` would overflow on the D2H copy
    with pytest.raises(ValueError):
        nt.polymul_rns_batch(A.cpu(), Bm.cpu(), basis,
                             out=torch.empty(A.shape, dtype=torch.int32))


def test_pair_cache_is_bounded_and_weak():
    plan = nt.build_plan(1 << 10, bits=40, seed=0)
    x = dev(rand(plan.q, plan.n, 5))
    before = len(K._PAIRS)
    tw = plan.tw_fwd.clone()  # a foreign device table
    y = x.clone()
    K.ntt_ct(y, tw, *plan.red_args, False, None)
    assert len(K._PAIRS) == before + 1
    z = x.clone()
    K.ntt_ct(z, plan.tw_fwd, *plan.red_args, False, None)
    assert torch.equal(y, z)
    del tw
    gc.collect()
    assert len(K._PAIRS) == before  # evicted with its table
    # numpy tables: paired once, reused while unchanged, re-paired after an edit
    tw_h = plan.tw_fwd.cpu().numpy().copy()
    p1, _ = K._pairs_for(tw_h, plan.q)
    p2, _ = K._pairs_for(tw_h, plan.q)
    assert p1 is p2
    tw_h[3] ^= 1
    p3, _ = K._pairs_for(tw_h, plan.q)
    assert p3 is not p1 and int(p3[3, 0]) == int(tw_h[3])
    for _ in range(K._PAIRS_MAX + 8):
        K._pairs_for(plan.tw_fwd.clone(), plan.q)
    assert len(K._PAIRS) <= K._PAIRS_MAX


def test_mixed_variant_basis_matches_oracle():
    n = 1 << 13
    primes = nt.RnsBasis.build(n, 60, 4, seed=0).primes
    plans = [nt.build_plan(n, q, seed=0, variant=v)
             for q, v in zip(primes, ["proposed", "classical", "dhem", "builtin"])]
    basis = nt.RnsBasis.from_plans(plans)
    assert basis.device_variant == "proposed"
    A, Bm = _batch(basis, 2, 7), _batch(basis, 2, 70)
    got = nt.polymul_rns_batch(dev(A), dev(Bm), basis).cpu().numpy()
    want = oracle.polymul_rns(A, Bm, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)


def test_device_caches_keyed_by_device():
    basis = nt.RnsBasis.build(1 << 12, 50, 2, seed=0)
    fwd, _, _ = basis.device_tables()
    key = ("tables", torch.cuda.current_device())
    assert key in basis._dev and basis._dev[key][0] is fwd
    assert basis.plans[0].tables_ready
    assert basis.plans[0].fwd_pairs.device == torch.device("cuda", torch.cuda.current_device())


def test_concurrent_host_threads_on_split_path():
    """Two host threads multiply different batches at the same time through
    the two-stream split (>= 128 limb-products) and the host pipeline: the
    fork/join events and copy streams are per host thread, so neither call
    waits on - or reads - the other's data (capi.cu shared
    per-device events)."""
    import threading

    basis = nt.RnsBasis.build(1 << 14, 60, 8, seed=0)
    batches = [(_batch(basis, 17, 100 * k), _batch(basis, 17, 100 * k + 50)) for k in range(2)]
    want = [nt.polymul_rns_batch(dev(a), dev(b), basis).cpu().numpy() for a, b in batches]
    got = [None, None]
    errors = []

    def work(k):
        try:
            torch.cuda.set_device(0)
            a, b = batches[k]
            for _ in range(5):
                da, db = dev(a), dev(b)
                dev_out = nt.polymul_rns_batch(da, db, basis)
                host_out = nt.polymul_rns_batch(a, b, basis)
                torch.cuda.synchronize()
                if not (np.array_equal(dev_out.cpu().numpy(), want[k]) and
                        np.array_equal(np.asarray(host_out), want[k])):
                    errors.append(k)
            got[k] = dev_out.cpu().numpy()
        except Exception as exc:  # noqa: BLE001 - reported below
            errors.append(repr(exc))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


def test_transform_fast_path_tracks_twiddle_edits():
    """The transforms' fast path (pair table attached to the plan's device
    twiddle tensor) must notice an in-place edit of that tensor: after
    overwriting tw_fwd with another prime's table the result follows the
    new table, and restoring it restores the original result."""
    n = 1 << 14
    p1 = nt.build_plan(n, bits=60, seed=1)
    x0 = rand(p1.q, n, 3)
    f, _ = oracle.twiddles(p1.q, p1.psi, 14)
    want = x0.copy()
    oracle.ntt_ct(want, f, *p1.red_args, False)
    x = torch.from_numpy(x0.copy()).cuda()
    nt.kernels.ntt_ct(x, p1.tw_fwd, *p1.red_args, False, None)
    assert np.array_equal(x.cpu().numpy(), want)
    saved = p1.tw_fwd.clone()
    p1.tw_fwd.copy_(p1.tw_inv)  # a different (inverse) table, same prime
    other = x0.copy()
    oracle.ntt_ct(other, p1.tw_inv.cpu().numpy(), *p1.red_args, False)
    x = torch.from_numpy(x0.copy()).cuda()
    nt.kernels.ntt_ct(x, p1.tw_fwd, *p1.red_args, False, None)
    assert np.array_equal(x.cpu().numpy(), other)
    p1.tw_fwd.copy_(saved)
    x = torch.from_numpy(x0.copy()).cuda()
    nt.kernels.ntt_ct(x, p1.tw_fwd, *p1.red_args, False, None)
    assert np.array_equal(x.cpu().numpy(), want)
