"""Multi-GPU sharding of the polymul hot path (one process per GPU).

Every (ciphertext, limb) product is independent (reference rns.py:116-119,
polymul.py:187-203), so the path shards with NO data-path collective:

* by ciphertext (BASELINE cfg3): rank r owns a contiguous, balanced span of
  the batch and runs ``polymul_rns_batch`` on it - weak scaling;
* by limb (BASELINE cfg4, 32 limbs over 8 GPUs): rank r owns a contiguous
  span of the basis (``sub_basis``) and only that span's twiddle tables.

Results stay sharded.  ``gather`` (an all-gather over torch.distributed:
NCCL on GPUs, gloo in the CPU tests) reassembles them off the timed path
when one rank needs the whole product.
"""

from __future__ import annotations

import torch

from .rns import RnsBasis


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous [lo, hi) of ``total`` units owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    if total < 0:
        raise ValueError("total < 0")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def sub_basis(basis: RnsBasis, world: int, rank: int) -> tuple[RnsBasis, int, int]:
    """The limb span of ``rank`` as its own basis (cfg4 limb sharding)."""
    lo, hi = shard_range(basis.num_limbs, world, rank)
    if hi <= lo:
        raise ValueError(f"rank {rank} owns no limbs ({basis.num_limbs} over {world})")
    return RnsBasis.from_plans(basis.plans[lo:hi]), lo, hi


def gather(shard: torch.Tensor, total: int, dim: int = 0, group=None) -> torch.Tensor:
    """All-gather uneven contiguous shards along ``dim`` (off the hot path).

    uint64 travels bit-reinterpreted as int64 (collectives do not reduce it,
    only move it).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_range(total, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    x = shard.movedim(dim, 0)
    payload = x.view(torch.int64) if x.dtype == torch.uint64 else x
    padded = torch.zeros((width, *payload.shape[1:]), dtype=payload.dtype,
                         device=payload.device)
    padded[: payload.shape[0]] = payload
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded.contiguous(), group=group)
    parts = [b[: hi - lo] for b, (lo, hi) in zip(bufs, sizes)]
    out = torch.cat(parts, 0)
    if x.dtype == torch.uint64:
        out = out.view(torch.uint64)
    return out.movedim(0, dim)
