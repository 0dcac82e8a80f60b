"""GQA comparison variant on the B200 decode kernels (attnkit/decode.py:232-240, :258-261).

The reference's non-latent ``attend_local`` branch for ``gqa``: every query head i reads
KV slot ``i // (h/g)`` (``kv_map``, zoo.py:35-38) of the post-RoPE key stream ``k`` and the
value stream ``v`` (zoo.py:47-58), logits are ``tau * q . K^T`` with tau = 1/sqrt(d_h)
(config.py:112), softmax, output ``P . V``. On the GPU it runs on the same split-KV kernel as
MLRA/MLA (K2, GQA instantiation: per KV head one K and one V sub-block per tile) followed by
the split merge; there is nothing to absorb and nothing to up-project.

``GqaDecodeEngine`` is the batched serving path (the MLA/GQA comparison rows of the
benchmark); ``attend_local_gqa`` / ``absorbed_decode_step_gqa`` are the drop-in functions
``decode.attend_local`` / ``decode.absorbed_decode_step`` route to for ``cfg.variant == "gqa"``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .cache import GqaLayout, PagedCache, PagedLatentCache
from .config import AttnConfig
from .errors import ConfigError, RoutingError

LOG2E = 1.4426950408889634


def _check_gqa(cfg: AttnConfig) -> None:
    if cfg.variant != "gqa":
        raise RoutingError(f"GQA decode path called for variant {cfg.variant!r}")


def gqa_layout(cfg: AttnConfig, own) -> GqaLayout:
    return GqaLayout(len(own.kv_slots), cfg.d_h)


def _local_groups(cfg: AttnConfig, own) -> tuple[int, int]:
    """(G local KV heads, R query heads per local KV head); the owned heads must be the
    contiguous head blocks of the owned slots (what tpsim.py:58-131 assigns)."""
    heads, slots = list(own.heads), list(own.kv_slots)
    G = len(slots)
    if G == 0 or len(heads) % G:
        raise ConfigError(f"gqa: {len(heads)} heads do not split over {G} KV slots")
    R = len(heads) // G
    reps = cfg.h // cfg.g
    for i, head in enumerate(heads):
        if head // reps != slots[i // R]:
            raise ConfigError("gqa: owned heads must be grouped by owned KV slot in order")
    return G, R


def queries_to_device(cfg: AttnConfig, layout: GqaLayout, q, heads, G: int, R: int, device) -> torch.Tensor:
    """[.., h, d_h] queries -> this device's [B, G, R, dhp] bf16 (zero-padded)."""
    qt = torch.as_tensor(np.asarray(q) if not torch.is_tensor(q) else q, dtype=torch.float32, device=device)
    if qt.dim() == 2:
        qt = qt[None]
    qt = qt[:, list(heads)]
    out = torch.zeros((qt.shape[0], G, R, layout.dhp), dtype=torch.float32, device=device)
    out[..., :cfg.d_h] = qt.reshape(qt.shape[0], G, R, cfg.d_h)
    return out.to(torch.bfloat16).contiguous()


def score_scale(cfg: AttnConfig) -> float:
    return float(cfg.tau) * LOG2E


def attend_local_gqa(cfg: AttnConfig, own, cache: PagedLatentCache, queries: dict) -> list:
    """Per-head contributions of one computing unit (decode.py:232-240): one per owned head."""
    _check_gqa(cfg)
    if cache.n == 0:
        raise ConfigError("cache read: stream 'k' is empty")
    if "q" not in queries:
        raise ConfigError("gqa attend_local needs queries['q'] (h, d_h)")
    G, R = _local_groups(cfg, own)
    layout = cache.layout
    pc = cache.paged
    q = queries_to_device(cfg, layout, queries["q"], own.heads, G, R, pc.device)
    nsplit = ops.gqa_default_splits(1, G, max(cache.n, 1))
    ws = ops.GqaWorkspace(1, G, R, layout.dhp, nsplit, pc.device)
    out = ops.gqa_decode_step(q, pc.pool, pc.block_table, pc.seqlens, pc.page_size, nsplit, score_scale(cfg), ws)
    ops.check_status(ws.status, "softmax_rows")  # NaN / no finite logit -> NumericError (tensors.py:74-78)
    cache.reads += cache.n * cache.row_elements()
    vecs = out[0, :, :cfg.d_h].double().cpu().numpy()
    return [(head, vecs[j]) for j, head in enumerate(own.heads)]


class GqaDecodeEngine:
    """Batched GQA decode attention for one device: B sequences in one paged pool.

    ``own`` = this device's heads and KV slots (full ownership = TP1; ``tp.shard_ownership``
    otherwise). ``decode_attention`` = K2 (GQA) + split merge -> fp32 [B, h_local, d_h].
    """

    def __init__(self, cfg: AttnConfig, own=None, *, batch: int, max_tokens: int, page_size: int = 128,
                 device=None, nsplit: int | None = None, page_order=None):
        from .decode import full_ownership

        _check_gqa(cfg)
        self.cfg = cfg
        self.own = own or full_ownership(cfg)
        self.G, self.R = _local_groups(cfg, self.own)
        self.layout = gqa_layout(cfg, self.own)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.heads = list(self.own.heads)
        self.cache = PagedCache(self.layout, batch, max_tokens, page_size, self.device, page_order)
        self.scale = score_scale(cfg)
        self.nsplit = nsplit or ops.gqa_default_splits(batch, self.G, max_tokens)
        self.workspace = ops.GqaWorkspace(batch, self.G, self.R, self.layout.dhp, self.nsplit, self.device)
        self.out = torch.empty((batch, self.G * self.R, self.layout.dhp), dtype=torch.float32, device=self.device)

    @property
    def batch(self) -> int:
        return self.cache.batch

    def prepare_queries(self, q) -> torch.Tensor:
        """[B, h, d_h] (any float, host or device) -> this device's [B, G, R, dhp] bf16."""
        return queries_to_device(self.cfg, self.layout, q, self.heads, self.G, self.R, self.device)

    def check_numeric(self) -> None:
        """NumericError if any step since the last check flagged a NaN / non-finite softmax row."""
        ops.check_status(self.workspace.status, "softmax_rows")

    def decode_attention(self, q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """One decode-attention step: [B, G, R, dhp] bf16 -> fp32 [B, h_local, d_h] (a view
        of the padded [B, h_local, dhp] output when d_h < dhp)."""
        c = self.cache
        res = ops.gqa_decode_step(q, c.pool, c.block_table, c.seqlens, c.page_size, self.nsplit, self.scale,
                                  self.workspace, out=self.out if out is None else out)
        return res[..., :self.cfg.d_h]
