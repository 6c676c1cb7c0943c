"""Multi-GPU plumbing: one process per GPU, one NCCL communicator per process.

The engine itself calls NCCL (all-reduce of epoch counts, all-gather of
deterministic events) on its own streams; torch.distributed is only used to
ship the 128-byte NCCL unique id from rank 0 to the other ranks.

    comm = Comm.from_torch_distributed(device=local_rank)   # inside torchrun
    cfg = adsamp.EngineConfig(..., comm=comm)
    res = kadabra.estimate_bc(graph, eps, delta, cfg)        # same result on every rank
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib


class Comm:
    def __init__(self, nranks: int, rank: int, unique_id: bytes, device: int = -1):
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self._h = C.c_void_p()
        check(lib().adsb_comm_init(nranks, rank, buf, device, C.byref(self._h)))
        self.nranks, self.rank, self.device = nranks, rank, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().adsb_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, device: int = -1) -> "Comm":
        """Create the communicator for the current torch.distributed group."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = cls.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0)
        return cls(world, rank, bytes(t.cpu().tolist()), device)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().adsb_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
