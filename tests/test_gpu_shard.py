"""Multi-rank path through the CUDA kernels.  Only one GPU is reachable, so
two ranks share it and talk over gloo: each rank multiplies ITS shard of a
[B, L, n] batch with the sm_100a kernels (by ciphertext, and by limb with
only its own limbs' tables via ``shard.sub_basis``), the shards are
gathered, and rank 0 compares the whole product with the C oracle.  Then
``bench.py --gpus 2`` (no outer launcher) spawns its own ranks and reports
n_gpus 2 for both partitions."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import rand

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, log_n, L, A, Bm, out_q):
    sys.path.insert(0, ROOT)
    import paper_2209_01290_b200 as nt
    from paper_2209_01290_b200.shard import gather, shard_range, sub_basis

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        full = nt.RnsBasis.build(1 << log_n, 60, L, seed=0)
        B = A.shape[0]
        if mode == "ct":
            lo, hi = shard_range(B, world, rank)
            c = nt.polymul_rns_batch(torch.from_numpy(A[lo:hi]).cuda(),
                                     torch.from_numpy(Bm[lo:hi]).cuda(), full)
            whole = gather(c.cpu(), B, dim=0)
        else:
            sb, lo, hi = sub_basis(full, world, rank)
            fwd, _, _ = sb.device_tables()
            assert fwd.shape[0] == hi - lo  # only this rank's limbs are resident
            a = torch.from_numpy(np.ascontiguousarray(A[:, lo:hi])).cuda()
            b = torch.from_numpy(np.ascontiguousarray(Bm[:, lo:hi])).cuda()
            c = nt.polymul_rns_batch(a, b, sb)
            whole = gather(c.cpu(), L, dim=1)
        if rank == 0:
            out_q.put(whole.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,log_n,L,B", [("ct", 14, 3, 5), ("limb", 14, 5, 2),
                                            ("ct", 16, 2, 3), ("limb", 17, 3, 1)])
def test_world2_shards_through_kernels(mode, log_n, L, B):
    import paper_2209_01290_b200 as nt

    n = 1 << log_n
    basis = nt.RnsBasis.build(n, 60, L, seed=0)
    A = np.stack([np.stack([rand(q, n, 7 * b + l) for l, q in enumerate(basis.primes)])
                  for b in range(B)])
    Bm = np.stack([np.stack([rand(q, n, 501 + 7 * b + l) for l, q in enumerate(basis.primes)])
                   for b in range(B)])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, log_n, L, A, Bm, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = oracle.polymul_rns(A, Bm, basis.primes, [p.psi for p in basis.plans])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("shard", ["ct", "limb"])
def test_bench_self_spawns_two_ranks(shard):
    env = dict(os.environ, NTTB_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--log-n", "14", "--limbs", "8", "--batch", "4",
           "--shard", shard, "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["parity"]["ok"] is True
    assert rec["scaling"] == ("weak" if shard == "ct" else "strong")
    assert rec["config"]["parallelism"].startswith(
        "shard-by-ciphertext" if shard == "ct" else "shard-by-limb")
    assert rec["roofline"]["per_rank_products_per_step"] == (4 * 8 if shard == "ct" else 4 * 4)
