"""Replica sharding across GPUs.

Replicas are independent (md.py:243-273) and the noise stream is keyed by
(seed, global replica index, step) (md.py:127-131), so rank g of G simply
owns a contiguous block of global replica indices and passes its first
index as `rep_offset`; no per-step collective exists.  The only
communication is an end-of-run gather of per-replica observables and final
states over torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations


def replica_shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first global replica, count) owned by `rank`; the first total % world
    ranks get one extra replica, so any total works."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def gather_replicas(local, total: int, group=None):
    """All-gather a [R_local, ...] tensor into [total, ...] in global replica
    order (variable shard sizes padded to the largest)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [replica_shard(total, world, r)[1] for r in range(world)]
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])
