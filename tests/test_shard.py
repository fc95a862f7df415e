"""N>1 plumbing on CPU: the balanced partition, and world_size-2 gloo
processes reassembling uneven shards with ``shard.gather`` along the
ciphertext and the limb dimension (plain uint64 data - the GPU test
tests/test_gpu_shard.py runs the same sharding through the CUDA kernels)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_01290_b200.shard import gather, shard_range


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


def _worker(rank, world, port, full, dim, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(full.shape[dim], world, rank)
        mine = np.ascontiguousarray(np.take(full, range(lo, hi), axis=dim))
        got = gather(torch.from_numpy(mine), full.shape[dim], dim=dim)
        if rank == 0:
            out_q.put(got.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,shape", [(0, (5, 3, 16)), (1, (2, 21, 8)), (1, (3, 3, 4))])
def test_gloo_world2_gather_uneven(dim, shape):
    rng = np.random.default_rng(3)
    full = rng.integers(0, 2**64, size=shape, dtype=np.uint64)
    full[..., 0] = np.uint64(2**64 - 1)  # top bit set: survives the int64 view
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, full, dim, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got.dtype == np.uint64 and np.array_equal(got, full)
