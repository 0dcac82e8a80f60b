"""Attention output side of one tensor-parallel rank.

Reference: ``attnkit/zoo.py:125-127`` (gated_output: ``out_flat * sigmoid(hidden @ w_g)``) and
the attention half of ``zoo.py:130-152`` (block_forward: ``hidden + gated @ w_o``). The
reference has no tensor-parallel output side; the decode path sums per-device attention
contributions in device order (``decode.py:264-285``, ``tpsim.py:249-286``). Because the gate
and W^O are linear in the attention output, a rank applies them to what it holds -- its heads
(MLA / GQA / GLA sharding) or a per-head partial of every head (MLRA-4 by branch) -- and the
ranks' [B, d] results are summed once:

    y = hidden + sum_r (attn_r * sigmoid(hidden @ W_g[:, cols_r])) @ W_o[cols_r, :]

``OutputProjection`` runs that per rank as K4a (gate + bf16 cast of the attention output) and
K4 (``mlra_outproj``): the W^O GEMM on tensor cores fused with a one-shot all-reduce over peer
memory (every rank stores its slab partials into every peer's communication region and sums
the world partials in rank order) -- no NCCL call. ``TpComm`` sets the regions up: a dedicated allocation per rank, CUDA IPC handles
exchanged over the process group (any backend), peers opened with lazy peer access.

The gate pre-activation ``hidden @ W_g`` depends on the block input only; it is computed on
the pre-attention side (a cuBLAS GEMM next to the query projections), not here.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .collective import PeerRegions
from .errors import ConfigError, ShapeMismatchError

__all__ = ["TpComm", "OutputProjection"]


class TpComm(PeerRegions):
    """Communication regions of a process group for K4 (one per rank, mapped in every rank)."""

    def __init__(self, group, batch: int, d: int, device=None):
        import torch.distributed as dist

        self.batch, self.d = int(batch), int(d)
        super().__init__(group, ops.outproj_comm_bytes(batch, d, dist.get_world_size(group)), device)


def _head_columns(heads, d_h: int) -> np.ndarray:
    return np.concatenate([np.arange(i * d_h, (i + 1) * d_h) for i in heads])


class OutputProjection:
    """K4 for one rank: its W_o rows (bf16) and W_g columns, optional TpComm for world > 1."""

    def __init__(self, cfg, w, heads, *, batch: int, device=None, comm: TpComm | None = None):
        self.cfg = cfg
        self.heads = list(heads)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        tensors = getattr(w, "tensors", w)
        if "w_o" not in tensors:
            raise ConfigError("output projection needs w_o (attnkit/weights.py:100)")
        cols = _head_columns(self.heads, cfg.d_h)
        w_o = np.asarray(tensors["w_o"])
        if w_o.shape != (cfg.out_flat_dim, cfg.d):
            raise ShapeMismatchError(f"w_o {w_o.shape} != {(cfg.out_flat_dim, cfg.d)}")
        self.w_o = torch.tensor(w_o[cols], dtype=torch.float32).to(self.device, torch.bfloat16).contiguous()
        self.w_g = None
        if cfg.gated:
            if "w_g" not in tensors:
                raise ConfigError("gated config without w_g (attnkit/weights.py:98-99)")
            self.w_g = torch.tensor(np.asarray(tensors["w_g"])[:, cols], dtype=torch.float32, device=self.device)
        self.batch = int(batch)
        self.comm = comm
        if comm is not None and (comm.batch != self.batch or comm.d != cfg.d):
            raise ConfigError("TpComm was sized for another batch / model width")
        self.y = torch.empty((self.batch, cfg.d), dtype=torch.float32, device=self.device)
        self.workspace = ops.outproj_workspace(self.batch, self.width, self.device)

    @property
    def width(self) -> int:
        return len(self.heads) * self.cfg.d_h

    def gate_pre(self, hidden: torch.Tensor) -> torch.Tensor | None:
        """hidden @ W_g[:, this rank's columns] (pre-attention side; fp32)."""
        return None if self.w_g is None else (hidden.float() @ self.w_g).contiguous()

    def __call__(self, attn: torch.Tensor, hidden: torch.Tensor, gate_pre: torch.Tensor | None = None,
                 residual: bool = True, out: torch.Tensor | None = None) -> torch.Tensor:
        """attn [B, h_local, d_h] (or [B, h_local*d_h]) fp32, hidden [B, d] fp32 -> y [B, d]."""
        B = attn.shape[0]
        if self.comm is not None and self.comm.world > 1 and B != self.comm.batch:
            # K4 lays out the receive slots, flags and epoch counter of the region from the
            # call's batch: a call of another batch would read the counters at the wrong place
            raise ConfigError(f"multi-rank output projection sized for batch {self.comm.batch}, called with {B}")
        a = attn.reshape(B, -1)
        if a.shape[1] != self.width:
            raise ShapeMismatchError(f"attention width {a.shape[1]} != {self.width} ({len(self.heads)} heads)")
        if gate_pre is None and self.w_g is not None:
            gate_pre = self.gate_pre(hidden)
        y = self.y[:B] if out is None else out
        resid = hidden.float().contiguous() if residual else None
        if self.comm is None or self.comm.world == 1:
            return ops.outproj(a.contiguous(), gate_pre, self.w_o, resid, y, workspace=self.workspace)
        return ops.outproj(a.contiguous(), gate_pre, self.w_o, resid, y, self.comm.rank, self.comm.world,
                           self.comm.ptrs, workspace=self.workspace)
