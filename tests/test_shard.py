"""N>1 path on CPU: world_size-2 gloo processes shard a [B, L, n] RNS batch by
ciphertext and by limb, compute their shards (the C oracle stands in for the
GPU kernel here - CPU test), and gather; the result must equal the unsharded
product.  Also unit-tests the balanced partition."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_01290_b200.shard import gather, shard_range, sub_basis


def test_shard_range_partitions():
    for total in (0, 1, 7, 21, 32, 168):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, A, Bm, primes, psis, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_2209_01290_b200 as nt

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, L, n = A.shape
        if mode == "ciphertext":
            lo, hi = shard_range(B, world, rank)
            mine = oracle.polymul_rns(A[lo:hi], Bm[lo:hi], primes, psis)
            full = gather(torch.from_numpy(mine), B, dim=0)
        else:  # limb sharding (cfg4 layout): rank owns limbs [lo, hi)
            basis = nt.RnsBasis.from_plans(
                [nt.params._plan_from_root(n, nt.Modulus(q), psi, "proposed")
                 for q, psi in zip(primes, psis)])
            sb, lo, hi = sub_basis(basis, world, rank)
            assert list(sb.primes) == primes[lo:hi]
            mine = oracle.polymul_rns(A[:, lo:hi], Bm[:, lo:hi], primes[lo:hi], psis[lo:hi])
            full = gather(torch.from_numpy(np.ascontiguousarray(mine)), L, dim=1)
        if rank == 0:
            out_q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["ciphertext", "limb"])
def test_gloo_world2_sharded_equals_whole(mode):
    import oracle

    rng = np.random.default_rng(3)
    primes = [1152921504606584833, 1152921504606748673, 1152921504606830593]
    n, B = 64, 5
    import paper_2209_01290_b200 as nt

    psis = [nt.find_primitive_root(q, 2 * n, 0) for q in primes]
    A = np.stack([np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in primes])
                  for _ in range(B)])
    Bm = np.stack([np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in primes])
                   for _ in range(B)])
    want = oracle.polymul_rns(A, Bm, primes, psis)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, A, Bm, primes, psis, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, want)
