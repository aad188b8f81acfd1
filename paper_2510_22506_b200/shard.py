"""Mode-0 sharding of the sweep across GPUs, one process per GPU.

``Shard(rank, nranks, backend)`` is passed to ``run(..., shard=...)``:

* ``backend="nccl"`` (production): rank 0 makes an NCCL unique id, it is
  broadcast with ``torch.distributed`` (any backend), and the library runs
  its collectives with NCCL on its own CUDA stream (``fctn_set_comm``).
* ``backend="host"`` (tests): the library stages its few collective payloads
  through host memory and calls back into ``torch.distributed`` (gloo), so
  ranks can share one GPU without kernels that wait on each other
  (``fctn_set_comm_host``).

Only the collectives' transport differs; the decomposition is the same:
X and the mask are split into the standard slabs of mode 0, factors / solves
/ Gram network are replicated, Y_k (k != 0) is all-reduced, Y_0's rows are
all-gathered, the four sweep sums are all-reduced.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = ["Shard"]


@dataclass
class Shard:
    rank: int
    nranks: int
    backend: str = "nccl"
    group: object = None

    def slab(self, I0: int):
        return _native.slab_of(I0, self.rank, self.nranks)

    def attach(self, ctx: "_native.Context"):
        import torch
        import torch.distributed as dist

        if self.backend == "nccl":
            obj = [_native.nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=self.group)
            ctx.set_comm_nccl(obj[0], self.rank, self.nranks)
        elif self.backend == "host":
            group = self.group
            nranks = self.nranks

            def allreduce(a: np.ndarray):
                t = torch.from_numpy(a)
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

            def allgather(a: np.ndarray) -> np.ndarray:
                t = torch.from_numpy(a)
                out = [torch.empty_like(t) for _ in range(nranks)]
                dist.all_gather(out, t, group=group)
                return torch.cat(out).numpy()

            ctx.set_comm_host(allreduce, allgather, self.rank, self.nranks)
        else:
            raise ValueError(f"unknown shard backend {self.backend!r}")
