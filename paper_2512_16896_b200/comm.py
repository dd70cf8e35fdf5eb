"""Native shard communicator (sb_comm_*, include/scenebatch_b200.h): the engine's
multi-GPU exchange without PyTorch. One process per GPU; a TCP star through rank 0 for the
bootstrap and host values, CUDA-IPC-mapped count boards in HBM for the device exchange the
FIFO fast path chains its rounds on."""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional

from . import _capi as A


def default_endpoint() -> tuple:
    """(host, port) of the rendezvous: SB_COMM_ADDR / SB_COMM_PORT, else torchrun's
    MASTER_ADDR and MASTER_PORT + 1 (the agent store keeps MASTER_PORT itself)."""
    host = os.environ.get("SB_COMM_ADDR", os.environ.get("MASTER_ADDR", "127.0.0.1"))
    if "SB_COMM_PORT" in os.environ:
        return host, int(os.environ["SB_COMM_PORT"])
    return host, int(os.environ.get("MASTER_PORT", "29500")) + 1


class Comm:
    """sb_comm: rank `rank` of `world_size` processes. device=None: host exchange only."""

    def __init__(self, rank: int, world_size: int, device: Optional[int] = 0,
                 host: Optional[str] = None, port: Optional[int] = None, timeout_s: float = 300.0):
        dh, dp = default_endpoint()
        h = C.c_void_p()
        A.check(A.lib().sb_comm_create(rank, world_size, -1 if device is None else device,
                                       (host or dh).encode(), port or dp, timeout_s, C.byref(h)))
        self._h = h
        self.rank, self.world_size, self.device = rank, world_size, device

    def close(self) -> None:
        if self._h:
            A.lib().sb_comm_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard(self, n_total: int) -> "CommShard":
        """This rank's contiguous variation range of n_total + the comm's callbacks."""
        s = A.sb_shard()
        A.check(A.lib().sb_comm_shard(self._h, n_total, C.byref(s)))
        return CommShard(self, s)

    def allgather(self, vals: List[int]) -> List[int]:
        n = len(vals)
        send = (C.c_uint64 * max(1, n))(*[v & 0xFFFFFFFFFFFFFFFF for v in vals])
        recv = (C.c_uint64 * max(1, n * self.world_size))()
        A.check(A.lib().sb_comm_allgather(self._h, send, n, recv))
        return list(recv)[: n * self.world_size]

    def allgather_dev(self, send_ptr: int, n: int, recv_ptr: int, stream_ptr: int = 0) -> None:
        A.check(A.lib().sb_comm_allgather_dev(self._h, send_ptr, n, recv_ptr, stream_ptr))

    def barrier(self) -> None:
        A.check(A.lib().sb_comm_barrier(self._h))

    def uses_stream_waits(self) -> bool:
        return bool(A.lib().sb_comm_uses_stream_waits(self._h))


class CommShard:
    """Engine shard (same face as world.Shard) whose exchange runs inside the library."""

    def __init__(self, comm: Comm, s: "A.sb_shard"):
        self.comm = comm  # keeps the communicator alive as long as the shard
        self._s = s
        self.begin, self.end = int(s.begin), int(s.end)
        self.rank, self.world_size = int(s.rank), int(s.world_size)

    def to_c(self):
        return self._s
