"""Multi-GPU plumbing: one process per GPU, one communicator per process.

The engine runs its collectives (all-gather of per-sample increments, the
barrier variant's all-reduce of epoch counts, rank-invariant sizing) itself,
over one of two transports:

* NCCL (the product path over NVLink / NVSwitch); torch.distributed only
  ships the 128-byte NCCL unique id from rank 0 to the other ranks:

      comm = Comm.from_torch_distributed(device=local_rank)   # inside torchrun
      cfg = adsamp.EngineConfig(..., comm=comm)
      res = kadabra.estimate_bc(graph, eps, delta, cfg)        # same result on every rank

* host collectives over an existing torch.distributed group (e.g. gloo), for
  ranks that cannot form an NCCL communicator — several ranks on one GPU, or
  a CPU-only interconnect. The engine stages device buffers through pinned
  host memory and calls back into Python:

      comm = Comm.from_host_group(device=0)                     # gloo group, any GPU count
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (HOST_ALLGATHER_U64, HOST_ALLREDUCE_U32_SUM, HOST_ALLREDUCE_U64, HostCollectives, check, lib)


class Comm:
    def __init__(self, nranks: int, rank: int, unique_id: bytes, device: int = -1):
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self._h = C.c_void_p()
        check(lib().adsb_comm_init(nranks, rank, buf, device, C.byref(self._h)))
        self.nranks, self.rank, self.device = nranks, rank, device
        self.transport = "nccl"

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().adsb_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, device: int = -1) -> "Comm":
        """Create the NCCL communicator for the current torch.distributed group."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = cls.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0)
        return cls(world, rank, bytes(t.cpu().tolist()), device)

    @classmethod
    def from_host_group(cls, device: int = -1, group=None) -> "Comm":
        """Host-transport communicator over a CPU torch.distributed group (gloo)."""
        import torch
        import torch.distributed as dist
        self = cls.__new__(cls)
        self.rank, self.nranks, self.device = dist.get_rank(group), dist.get_world_size(group), device
        self.transport = "host"
        ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MAX, 2: dist.ReduceOp.MIN}

        def allreduce_u64(_user, buf, count, op):
            try:
                a = np.ctypeslib.as_array(buf, shape=(count,))
                t = torch.from_numpy(a.view(np.int64).copy())  # values < 2^63 (counts, sizes)
                dist.all_reduce(t, op=ops[op], group=group)
                a[:] = t.numpy().view(np.uint64)
                return 0
            except Exception:  # pragma: no cover - reported by the engine as a status
                return 1

        def allreduce_u32_sum(_user, buf, count):
            try:
                a = np.ctypeslib.as_array(buf, shape=(count,))
                t = torch.from_numpy(a.astype(np.int64))
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                a[:] = t.numpy().astype(np.uint32)
                return 0
            except Exception:  # pragma: no cover
                return 1

        def allgather_u64(_user, send, recv, count):
            try:
                s = torch.from_numpy(np.ctypeslib.as_array(send, shape=(count,)).view(np.int64).copy())
                out = [torch.empty_like(s) for _ in range(self.nranks)]
                dist.all_gather(out, s, group=group)
                r = np.ctypeslib.as_array(recv, shape=(count * self.nranks,))
                r[:] = torch.cat(out).numpy().view(np.uint64)
                return 0
            except Exception:  # pragma: no cover
                return 1

        # keep the ctypes thunks alive as long as the communicator
        self._ops = HostCollectives(HOST_ALLREDUCE_U64(allreduce_u64), HOST_ALLREDUCE_U32_SUM(allreduce_u32_sum),
                                    HOST_ALLGATHER_U64(allgather_u64))
        self._h = C.c_void_p()
        check(lib().adsb_comm_init_host(self.nranks, self.rank, device, C.byref(self._ops), None, C.byref(self._h)))
        return self

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().adsb_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
