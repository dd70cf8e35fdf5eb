"""Multi-GPU plumbing: one process per GPU, instances sharded into
contiguous variation ranges; the only exchange is the FIFO fast path's per-round survivor
counts and a relation placement's instance-0 anchor state (a few u64 per rank), done with
torch.distributed all_gather on the host values the engine already reads back."""
from __future__ import annotations

from typing import Callable, List


def shard_bounds(n_total: int, world: int) -> List[int]:
    """Contiguous variation ranges [b[r], b[r+1]) per rank (equal sizes up to one)."""
    return [n_total * r // world for r in range(world + 1)]


def torch_allgather(world: int) -> Callable[[List[int]], List[int]]:
    """sb_shard.allgather callback over the initialised torch.distributed group: every
    rank contributes the same number of u64 values; returns them rank-major."""
    import torch
    import torch.distributed as dist

    def allgather(vals: List[int]) -> List[int]:
        t = torch.tensor([v & 0xFFFFFFFFFFFFFFFF for v in vals], dtype=torch.uint64).view(torch.int64)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [int(v) & 0xFFFFFFFFFFFFFFFF for o in out for v in o.tolist()]

    return allgather
