"""Tensor parallelism for latent decode (replaces attnkit/tpsim.py).

Two levels:

* ``make_shards`` / ``sim_decode`` / ``ShardSet`` / ``TrafficLedger`` keep the reference's
  logical-device API (tpsim.py:147-286): every "device" is a separate cache + weight slice
  on the current GPU, attention runs on the B200 kernels per device, and the reduction is
  done in device-id order with the reduction kind asserted ("sum" for mlra, "concat"
  otherwise). The ledger's per-device read counts follow the same analytic rule as the
  reference (each owned stream read once per step).
* ``TPDecodeGroup`` is the real multi-GPU path: one process per GPU (torch.distributed),
  each rank holds the streams ``shard_ownership`` assigns it (MLRA-4 at TP4: one latent
  block + the replicated rotary key), computes its branch's alpha-scaled, up-projected
  output with K1+K2+K3, and one ``all_reduce(SUM)`` over the TP group produces the head
  outputs (the device-id-ordered sum of tpsim.py:275-276, up to fp reassociation). With
  more ranks than the TP degree the world is split into TP groups over disjoint batch
  slices (8 GPUs = 2 x TP4).

The sharding rule ``shard_ownership`` is the reference's (tpsim.py:58-131) for the served
variants.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .config import TP_DEGREES, AttnConfig
from .decode import (LatentUnit, Ownership, _check_served, _state, append_token_latent, attend_local, local_weights,
                     new_cache, reduce_contributions, token_projections)
from .errors import ConfigError, IntegrityError


def _ranges(total: int, parts: int, axis: str) -> list[tuple[int, ...]]:  # tpsim.py:51-55
    if parts <= 0 or total % parts != 0:
        raise ConfigError(f"cannot split {axis} of size {total} into {parts} shards")
    size = total // parts
    return [tuple(range(k * size, (k + 1) * size)) for k in range(parts)]


def shard_ownership(cfg: AttnConfig, phi: int, device_id: int) -> Ownership:  # tpsim.py:58-131
    if phi not in TP_DEGREES:
        raise ConfigError(f"unsupported TP degree {phi}; supported: {TP_DEGREES}")
    _check_served(cfg)
    h, k = cfg.h, device_id
    all_heads = tuple(range(h))
    if cfg.variant == "gqa":
        # KV-head axis first; beyond g devices, the query heads of one KV head are split
        g, r = cfg.g, h // cfg.g
        if phi <= g:
            slots = _ranges(g, phi, "KV-head axis")[k]
            return Ownership(tuple(range(slots[0] * r, (slots[-1] + 1) * r)), kv_slots=slots)
        per_group = phi // g
        if phi % g != 0 or r % per_group != 0:
            raise ConfigError(f"gqa: cannot split {r} heads per KV head across {per_group} devices")
        group = k // per_group
        heads = tuple(i + group * r for i in _ranges(r, per_group, "query-head axis")[k % per_group])
        return Ownership(heads, kv_slots=(group,))
    if cfg.variant == "mla":
        heads = _ranges(h, phi, "query-head axis")[k]
        return Ownership(heads, units=(LatentUnit(-1, -1, heads),))
    if cfg.variant == "gla":  # latent-group axis, then the heads of one group (tpsim.py:92-106)
        g, r = cfg.g, h // cfg.g
        if phi <= g:
            units = tuple(LatentUnit(j, -1, tuple(range(j * r, (j + 1) * r)))
                          for j in _ranges(g, phi, "latent-group axis")[k])
            return Ownership(tuple(i for u in units for i in u.heads), units=units)
        per_group = phi // g
        if phi % g != 0 or r % per_group != 0:
            raise ConfigError(f"gla: cannot split {r} heads per group across {per_group} devices")
        group = k // per_group
        heads = tuple(i + group * r for i in _ranges(r, per_group, "query-head axis")[k % per_group])
        return Ownership(heads, units=(LatentUnit(group, -1, heads),))
    if cfg.branches == 2:  # mlra-2: (group, block) units, group-first (tpsim.py:117-131)
        pairs = [(grp, b) for grp in range(2) for b in range(2)]
        half_heads = [tuple(range(grp * (h // 2), (grp + 1) * (h // 2))) for grp in range(2)]
        if phi == 1:
            return Ownership(all_heads, units=tuple(LatentUnit(grp, b, half_heads[grp]) for grp, b in pairs))
        if phi == 2:
            return Ownership(half_heads[k], units=tuple(LatentUnit(k, b, half_heads[k]) for b in range(2)))
        if phi == 4:
            grp, b = pairs[k]
            return Ownership(half_heads[grp], units=(LatentUnit(grp, b, half_heads[grp]),))
        grp, b = pairs[k // 2]
        heads = tuple(i + grp * (h // 2) for i in _ranges(h // 2, 2, "query-head axis")[k % 2])
        return Ownership(heads, units=(LatentUnit(grp, b, heads),))
    if phi <= 4:
        blocks = _ranges(4, phi, "latent-block axis")[k]
        return Ownership(all_heads, units=tuple(LatentUnit(-1, b, all_heads) for b in blocks))
    block, half = k // 2, k % 2
    heads = _ranges(h, 2, "query-head axis")[half]
    return Ownership(heads, units=(LatentUnit(-1, block, heads),))


def _resource_keys(own: Ownership) -> list[str]:  # tpsim.py:134-144 (latent family + gqa)
    if not own.units:
        return [f"{s}[{slot}]" for s in ("k", "v") for slot in own.kv_slots]
    return [unit.stream for unit in own.units] + ["rope"]


@dataclass
class DeviceShard:
    device_id: int
    own: Ownership
    cache: object
    attn_weights: dict

    @property
    def reads(self) -> int:
        return self.cache.reads


@dataclass
class TrafficLedger:  # tpsim.py:159-187
    variant: str
    phi: int
    d_h: int
    reads_per_step: list = field(default_factory=list)
    tokens_per_step: list = field(default_factory=list)
    replicated: dict = field(default_factory=dict)
    reduction: str = ""

    def per_token_loads(self, step: int = -1) -> list[Fraction]:
        tokens = self.tokens_per_step[step]
        return [Fraction(r, tokens * self.d_h) for r in self.reads_per_step[step]]

    def to_json_dict(self) -> dict:
        from .costs import fraction_str

        return {
            "variant": self.variant,
            "tp": self.phi,
            "reduction": self.reduction,
            "tokens_per_step": list(self.tokens_per_step),
            "reads_per_step": [list(r) for r in self.reads_per_step],
            "per_token_load_dh": [fraction_str(x) for x in self.per_token_loads()],
            "replicated": {k: list(v) for k, v in sorted(self.replicated.items())},
        }


class ShardSet:  # tpsim.py:190-246
    def __init__(self, cfg: AttnConfig, w, phi: int, pos_offset: int = 0):
        self.cfg, self.weights, self.phi, self.pos_offset = cfg, w, phi, pos_offset
        self.shards = []
        for device_id in range(phi):
            own = shard_ownership(cfg, phi, device_id)
            self.shards.append(DeviceShard(device_id, own, new_cache(cfg, own, pos_offset),
                                           local_weights(cfg, w, own)))
        self._check_coverage()
        resources: dict = {}
        for shard in self.shards:
            for key in _resource_keys(shard.own):
                resources.setdefault(key, []).append(shard.device_id)
        self.ledger = TrafficLedger(cfg.variant, phi, cfg.d_h,
                                    replicated={k: v for k, v in resources.items() if len(v) > 1},
                                    reduction="sum" if cfg.variant == "mlra" else "concat")

    def _check_coverage(self) -> None:
        expected = list(range(self.cfg.h))
        if self.cfg.variant == "mlra":
            per_head: dict = {}
            for s in self.shards:
                for unit in s.own.units:
                    for i in unit.heads:
                        per_head[i] = per_head.get(i, 0) + 1
            bad = {i: c for i, c in per_head.items() if c != self.cfg.branches}
            if sorted(per_head) != expected or bad:
                raise IntegrityError(f"mlra branch coverage wrong for heads {sorted(bad)}")
        elif sorted(i for s in self.shards for i in s.own.heads) != expected:
            raise IntegrityError("query heads not exactly covered by shards")

    @property
    def n(self) -> int:
        return self.shards[0].cache.n

    def __iter__(self):
        return iter(self.shards)

    def __len__(self):
        return len(self.shards)


def make_shards(cfg: AttnConfig, w, phi: int, pos_offset: int = 0) -> ShardSet:  # tpsim.py:249-250
    return ShardSet(cfg, w, phi, pos_offset)


def sim_decode(shards: ShardSet, h_t, order=None):  # tpsim.py:253-286
    """One distributed decode step over logical devices on the current GPU."""
    cfg, w = shards.cfg, shards.weights
    pos = shards.pos_offset + shards.n
    exec_order = list(order) if order is not None else list(range(len(shards)))
    if sorted(exec_order) != list(range(len(shards))):
        raise IntegrityError("execution order must visit every device exactly once")
    dev = shards.shards[0].cache.paged.device
    st = _state(cfg, w, dev)
    before = [s.cache.reads for s in shards.shards]
    by_device: dict = {}
    proj = None
    import torch

    if cfg.variant == "gqa":

        hidden = torch.as_tensor(np.asarray(h_t, dtype=np.float64).reshape(1, cfg.d), dtype=torch.float32, device=dev)
        q, k, v = st.projector(hidden, torch.tensor([pos], device=dev))
    for idx in exec_order:
        shard = shards.shards[idx]
        if cfg.variant == "gqa":
            slots = list(shard.own.kv_slots)
            rows = {"k": k[0][slots], "v": v[0][slots]}
            shard.cache.append_packed(shard.cache.layout.pack_rows(rows, device=dev)[None])
            by_device[shard.device_id] = attend_local(cfg, {}, shard.own, shard.cache,
                                                      {"q": q[0].double().cpu().numpy()})
            continue
        if proj is None:  # K-1 once per step (the ranks' replicated projections)
            proj = token_projections(cfg, st, h_t, pos)
            queries = {"q_nope": proj[2][0].double().cpu().numpy(), "q_rope": proj[3][0].double().cpu().numpy()}
        append_token_latent(cfg, st, shard.cache, proj[0], proj[1], pos, shard.own)  # fused K0 (owned blocks)
        by_device[shard.device_id] = attend_local(cfg, shard.attn_weights, shard.own, shard.cache, queries)
    contribs = [c for did in sorted(by_device) for c in by_device[did]]
    out, kind = reduce_contributions(cfg, contribs)
    if kind != shards.ledger.reduction:
        raise IntegrityError(f"{cfg.variant}: observed {kind!r} reduction, mechanism requires "
                             f"{shards.ledger.reduction!r}")
    shards.ledger.reads_per_step.append([s.cache.reads - b for s, b in zip(shards.shards, before)])
    shards.ledger.tokens_per_step.append(shards.n)
    return out, shards.ledger


# ----------------------------------------------------------------------------- real multi-GPU
def tp_layout(world_size: int, tp: int) -> tuple[int, int]:
    """(tp degree, data-parallel groups) for a world: TP groups of ``tp`` ranks over batch slices."""
    if world_size % tp:
        raise ConfigError(f"world size {world_size} is not a multiple of the TP degree {tp}")
    return tp, world_size // tp


def group_ranks(world_size: int, tp: int) -> list[list[int]]:
    """Contiguous rank groups: {0..tp-1}, {tp..2tp-1}, ... (topology-neutral on NVSwitch)."""
    _, dp = tp_layout(world_size, tp)
    return [list(range(g * tp, (g + 1) * tp)) for g in range(dp)]


class TPDecodeGroup:
    """One rank of a TP decode group (one process per GPU).

    ``compute(q_nope, q_rope) -> local`` is this rank's alpha-scaled, up-projected output for
    its owned units ([B, h_local, d_h] fp32; zeros elsewhere are implied by the layout); the
    group all-reduces (SUM) the full-head tensor. For mlra the local tensor covers all heads
    (every rank owns one block for every head); for mla the ranks own disjoint heads and the
    sum assembles them (the reference's "concat", expressed as a sum of disjoint supports).
    ``compute`` is injectable so the plumbing is testable on CPU with the gloo backend.
    """

    def __init__(self, cfg: AttnConfig, tp: int, rank: int, world_size: int, group=None, compute=None,
                 reducer=None):
        self.reducer = reducer  # collective.PeerAllReduce (K5, peer memory) or None (torch.distributed)
        self.cfg = cfg
        self.tp = tp
        self.rank = rank
        self.world_size = world_size
        self.tp_rank = rank % tp
        self.dp_index = rank // tp
        self.own = shard_ownership(cfg, tp, self.tp_rank)
        self.group = group
        self.compute = compute

    def batch_slice(self, batch: int) -> slice:
        _, dp = tp_layout(self.world_size, self.tp)
        per = batch // dp
        if per * dp != batch:
            raise ConfigError(f"global batch {batch} does not split over {dp} TP groups")
        return slice(self.dp_index * per, (self.dp_index + 1) * per)

    def step(self, q_nope, q_rope, full_out):
        """Run this rank's share and all-reduce into ``full_out`` [B_local, h, d_h] (in place)."""
        import torch.distributed as dist

        local = self.compute(q_nope, q_rope)
        heads = list(self.own.heads)
        if len(heads) == self.cfg.h:
            full_out.copy_(local)
        else:
            full_out.zero_()
            full_out[:, heads] = local
        if self.tp > 1:
            if self.reducer is not None:
                self.reducer(full_out)
            else:
                dist.all_reduce(full_out, op=dist.ReduceOp.SUM, group=self.group)
        return full_out


def reduction_kind(cfg: AttnConfig) -> str:
    return "sum" if cfg.variant == "mlra" else "concat"


def local_branch_reference(out_units: np.ndarray) -> np.ndarray:
    """Sum of per-unit contributions in ascending unit order (the reference's reducer order)."""
    return np.sum(out_units, axis=0)
