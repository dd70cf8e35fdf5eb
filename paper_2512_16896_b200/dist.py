"""Multi-GPU plumbing: one process per GPU, instances sharded into
contiguous variation ranges; the only exchange is the FIFO fast path's per-round survivor
counts and a relation placement's instance-0 anchor state (a few u64 per rank), done with
torch.distributed all_gather: over NCCL (NVLink / NVSwitch) when the process group has a
CUDA backend and a device is given, else over the CPU backend (gloo)."""
from __future__ import annotations

from typing import Callable, List


def shard_bounds(n_total: int, world: int) -> List[int]:
    """Contiguous variation ranges [b[r], b[r+1]) per rank (equal sizes up to one)."""
    return [n_total * r // world for r in range(world + 1)]


def torch_allgather(world: int, device=None) -> Callable[[List[int]], List[int]]:
    """sb_shard.allgather callback over the initialised torch.distributed group: every
    rank contributes the same number of u64 values; returns them rank-major. With `device`
    (a CUDA device of a group whose CUDA backend is NCCL) the values travel as one NCCL
    all_gather_into_tensor; otherwise as CPU tensors (gloo)."""
    import torch
    import torch.distributed as dist

    def allgather(vals: List[int]) -> List[int]:
        t = torch.tensor([v & 0xFFFFFFFFFFFFFFFF for v in vals], dtype=torch.uint64).view(torch.int64)
        if device is not None:
            src = t.to(device, non_blocking=False)
            out = torch.empty(world * len(vals), dtype=torch.int64, device=device)
            dist.all_gather_into_tensor(out, src)
            return [int(v) & 0xFFFFFFFFFFFFFFFF for v in out.cpu().tolist()]
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [int(v) & 0xFFFFFFFFFFFFFFFF for o in out for v in o.tolist()]

    return allgather


def init_group(local_rank: int):
    """One process per GPU: CPU tensors over gloo (timing reductions), CUDA tensors over
    NCCL (the engine's count exchange). Returns the CUDA device for torch_allgather, or None
    when only gloo could be initialised."""
    import torch
    import torch.distributed as dist

    if torch.cuda.is_available():
        try:
            dev = torch.device("cuda", local_rank)
            torch.cuda.set_device(dev)
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=dev)
            return dev
        except Exception:  # noqa: BLE001 -- fall back to the CPU backend alone
            if dist.is_initialized():
                dist.destroy_process_group()
    dist.init_process_group("gloo")
    return None


class _DevArray:
    """Zero-copy view of n u64 at a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def nccl_allgather_dev(world: int, device):
    """sb_shard.allgather_dev over the NCCL backend of the initialised group: the engine's
    device count words are gathered in place on the engine's stream (no host round trip)."""
    import torch
    import torch.distributed as dist

    def allgather_dev(send_ptr: int, n: int, recv_ptr: int, stream_ptr: int) -> None:
        src = torch.as_tensor(_DevArray(send_ptr, n), device=device).view(torch.int64)
        dst = torch.as_tensor(_DevArray(recv_ptr, world * n), device=device).view(torch.int64)
        with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr, device=device)):
            dist.all_gather_into_tensor(dst, src)

    return allgather_dev
