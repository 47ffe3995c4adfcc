"""Replica sharding across GPUs.

Replicas are independent (md.py:243-273) and the noise stream is keyed by
(seed, global replica index, step) (md.py:127-131), so rank g of G simply
owns a contiguous block of global replica indices and passes its first
index as `rep_offset`; no per-step collective exists.  The only
communication is an end-of-run gather of per-replica observables and final
states over torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


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


class ReplicaShards:
    """This rank's share of a replica-sharded run plus the few collectives
    the run needs, over torch.distributed (`group`, default the world).

    Tensors travel on the current CUDA device under NCCL and on the host
    under gloo (the CPU tests, and several ranks sharing one GPU); callers
    pass and receive host numpy arrays."""

    def __init__(self, total: int, group=None):
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized():
            raise RuntimeError("distributed=True needs an initialised torch.distributed "
                               "process group (one rank per GPU, e.g. torchrun)")
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.total = int(total)
        self.first, self.count = replica_shard(self.total, self.world, self.rank)
        if self.count == 0:
            raise ValueError(f"{self.total} replicas cannot be sharded over {self.world} ranks "
                             "(a rank would own none)")
        self.nccl = dist.get_backend(group) == "nccl"

    def _dev(self, t):
        import torch
        return t.to(torch.device("cuda", torch.cuda.current_device())) if self.nccl else t

    def gather(self, local):
        """[count, ...] host array -> [total, ...] in global replica order."""
        import torch
        out = gather_replicas(self._dev(torch.as_tensor(np.ascontiguousarray(local))),
                              self.total, self.group)
        return out.cpu().numpy()

    def min_int(self, x: int) -> int:
        import torch
        t = self._dev(torch.tensor([int(x)], dtype=torch.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def sum_int(self, xs):
        import torch
        t = self._dev(torch.tensor([int(x) for x in xs], dtype=torch.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().tolist()

    def barrier(self):
        self.dist.barrier(group=self.group)
