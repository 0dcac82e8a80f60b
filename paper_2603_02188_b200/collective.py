"""Collectives over NVLink peer memory for the tensor-parallel decode step.

The reference sums per-device contributions in device order (``attnkit/decode.py:264-285``,
``tpsim.py:275-276``). ``PeerAllReduce`` does that sum for the TP decode step's output with
K5 (``mlra_allreduce``): every rank stores its buffer into every peer's region and adds the
world copies in ascending rank order -- bit-identical results on all ranks, one kernel, no
NCCL call. ``PeerRegions`` sets the regions up for any process group: one dedicated
allocation per rank (``mlra_comm_alloc``), CUDA IPC handles exchanged with
``all_gather_object`` (works over gloo or NCCL groups), peers opened with lazy peer access.
"""

from __future__ import annotations

import torch

from . import ops

__all__ = ["PeerRegions", "PeerAllReduce"]


class PeerRegions:
    """One communication region per rank of `group`, mapped in this process (``ptrs[r]``)."""

    def __init__(self, group, nbytes: int, device=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nbytes = int(nbytes)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self.own = ops.comm_alloc(self.nbytes)
            handles = [None] * self.world
            dist.all_gather_object(handles, ops.ipc_handle(self.own), group=group)
            self.ptrs = [self.own if r == self.rank else ops.ipc_open(handles[r]) for r in range(self.world)]

    def close(self) -> None:
        if self.ptrs is None:
            return
        with torch.cuda.device(self.device):
            for r, p in enumerate(self.ptrs):
                if r != self.rank:
                    ops.ipc_close(p)
            ops.comm_free(self.own)
        self.ptrs = None


class PeerAllReduce(PeerRegions):
    """In-place-capable sum of an fp32 buffer of ``n`` values over the group (K5). Graph-safe:
    the call epoch lives in device memory. Every rank must issue the same calls."""

    def __init__(self, group, n: int, device=None):
        import torch.distributed as dist

        self.n = int(n)
        super().__init__(group, ops.allreduce_comm_bytes(self.n, dist.get_world_size(group)), device)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if x.numel() != self.n:
            raise ValueError(f"PeerAllReduce sized for {self.n} values, got {x.numel()}")
        return ops.allreduce(x, x if out is None else out, self.rank, self.world, self.ptrs)
