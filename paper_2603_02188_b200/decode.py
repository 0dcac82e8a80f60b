"""Drop-in decode API (attnkit/decode.py) backed by the B200 kernels.

Same names, argument meanings and error behaviour as the reference decode module:

* ``LatentUnit``, ``Ownership``, ``full_ownership``, ``owned_stream_layout``,
  ``new_cache`` (decode.py:31-103) -- ``new_cache`` returns a device-resident
  ``PagedLatentCache`` instead of a Python-list ``KvCache``;
* ``absorb_query`` (decode.py:155-167) -> kernel K1;
* ``local_weights`` (decode.py:190-199) -- the same (latent, heads, d_h) slices, plus a
  lazily built head-major bf16 device pack for K1/K3;
* ``attend_local`` (decode.py:204-230) -> K1 + K2 + K3 (per-unit up-projection);
* ``reduce_contributions`` (decode.py:264-285) -- host logic, unchanged;
* ``absorbed_decode_step`` / ``decode_step`` (decode.py:290-348) -> projections (torch),
  K0 append, K1 + K2 + K3 (branch sum and alpha_attn fused into K3).

``DecodeEngine`` is the batched serving path (many sequences, one paged pool) that the
benchmark drives. Every compute call requires CUDA and the built extension; there is no
CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .cache import GqaLayout, PagedCache, PagedLatentCache, RowLayout
from .config import LATENT_VARIANTS, AttnConfig
from .costs import calib_factors
from .errors import ConfigError, IntegrityError, RoutingError
from .projections import LatentProjector

SERVED = ("mla", "mlra", "gqa")


@dataclass(frozen=True)
class LatentUnit:
    """One latent slice and the heads it serves; -1 means axis not split (decode.py:31-41)."""

    group: int
    block: int
    heads: tuple

    @property
    def stream(self) -> str:
        return latent_stream_name(self.group, self.block)


@dataclass(frozen=True)
class Ownership:
    """What one computing unit holds: output heads plus cached-state slices (decode.py:44-50)."""

    heads: tuple
    kv_slots: tuple = ()
    units: tuple = ()


def latent_stream_name(group: int, block: int) -> str:  # attnkit/cache.py:147-155
    if group < 0 and block < 0:
        return "latent"
    if block < 0:
        return f"latent_{group}"
    if group < 0:
        return f"latent_b{block}"
    return f"latent_{group}_{block}"


def _check_served(cfg: AttnConfig) -> None:
    if cfg.variant not in SERVED:
        raise RoutingError(f"the B200 latent decode path serves {SERVED}; got {cfg.variant!r}")
    if cfg.variant == "mlra" and cfg.branches != 4:
        raise RoutingError("the B200 latent decode path serves the four-branch MLRA form (MLRA-4)")


def full_ownership(cfg: AttnConfig) -> Ownership:  # decode.py:53-76 (served variants)
    _check_served(cfg)
    all_heads = tuple(range(cfg.h))
    if cfg.variant == "gqa":
        return Ownership(all_heads, kv_slots=tuple(range(cfg.g)))
    if cfg.variant == "mla":
        return Ownership(all_heads, units=(LatentUnit(-1, -1, all_heads),))
    return Ownership(all_heads, units=tuple(LatentUnit(-1, b, all_heads) for b in range(4)))


def unit_width(cfg: AttnConfig) -> int:
    return cfg.d_c if cfg.variant == "mla" else cfg.block_dim


def row_layout(cfg: AttnConfig, own: Ownership):
    if cfg.variant == "gqa":
        return GqaLayout(len(own.kv_slots), cfg.d_h)
    return RowLayout(tuple(u.stream for u in own.units), unit_width(cfg), cfg.d_h_rope)


def owned_stream_layout(cfg: AttnConfig, own: Ownership) -> dict:  # decode.py:79-98
    return row_layout(cfg, own).row_shapes()


def new_cache(cfg: AttnConfig, own: Ownership | None = None, pos_offset: int = 0, *, device=None,
              page_size: int = 128, initial_tokens: int = 1024) -> PagedLatentCache:  # decode.py:101-103
    own = own or full_ownership(cfg)
    _check_served(cfg)
    return PagedLatentCache(cfg.variant, row_layout(cfg, own), pos_offset, device, page_size, initial_tokens)


# ----------------------------------------------------------------------------- weights
def _unit_weight_slices(cfg: AttnConfig, w, unit: LatentUnit) -> tuple[np.ndarray, np.ndarray]:
    """(latent, m, d_h) key/value up-projection slices (decode.py:170-187)."""
    heads = list(unit.heads)
    w_uk, w_uv = w["w_uk"], w["w_uv"]
    if unit.block >= 0:
        bs = cfg.block_dim
        w_uk = w_uk[unit.block * bs:(unit.block + 1) * bs]
        w_uv = w_uv[unit.block * bs:(unit.block + 1) * bs]
    d_lat = w_uk.shape[0]
    return (w_uk.reshape(d_lat, -1, cfg.d_h)[:, heads], w_uv.reshape(d_lat, -1, cfg.d_h)[:, heads])


class LocalWeights(dict):
    """``{"uk:<stream>": (latent, m, d_h), "uv:<stream>": ...}`` like decode.py:190-199, with a
    cached device pack: w_uk [m, d_h, NU*dlp] and w_uv [m, NU*dlp, d_h] (bf16, zero-padded)."""

    def packed(self, layout: RowLayout, device) -> tuple[torch.Tensor, torch.Tensor]:
        key = ("__packed__", layout, str(device))
        if key not in self.__dict__:
            uks = [np.asarray(self[f"uk:{u}"]) for u in layout.units]
            uvs = [np.asarray(self[f"uv:{u}"]) for u in layout.units]
            m, dh = uks[0].shape[1], uks[0].shape[2]
            nu, dlp, dl = layout.nb, layout.dlp, layout.dl
            uk = np.zeros((m, dh, nu * dlp), dtype=np.float32)
            uv = np.zeros((m, nu * dlp, dh), dtype=np.float32)
            for i, (a, b) in enumerate(zip(uks, uvs)):
                uk[:, :, i * dlp:i * dlp + dl] = np.transpose(a, (1, 2, 0))  # (lat, m, dh) -> (m, dh, lat)
                uv[:, i * dlp:i * dlp + dl, :] = np.transpose(b, (1, 0, 2))  # (lat, m, dh) -> (m, lat, dh)
            self.__dict__[key] = (torch.as_tensor(uk, device=device).to(torch.bfloat16).contiguous(),
                                  torch.as_tensor(uv, device=device).to(torch.bfloat16).contiguous())
        return self.__dict__[key]


def local_weights(cfg: AttnConfig, w, own: Ownership) -> LocalWeights:  # decode.py:190-199
    if cfg.variant not in LATENT_VARIANTS:
        return LocalWeights()
    out = LocalWeights()
    for unit in own.units:
        uk, uv = _unit_weight_slices(cfg, w, unit)
        out[f"uk:{unit.stream}"] = uk
        out[f"uv:{unit.stream}"] = uv
    return out


# ----------------------------------------------------------------------------- K1 as a function
def absorb_query(q_nope, w_uk, *, device=None) -> np.ndarray:
    """q~[i, c] = sum_p q_nope[i, p] W_uk[c, i, p] on the GPU (decode.py:155-167).

    ``w_uk`` is (latent, m*p) or (latent, m, p); returns float64 (m, latent) computed in
    bf16 inputs / fp32 accumulation by kernel K1.
    """
    q = np.asarray(q_nope, dtype=np.float64)
    m, p = q.shape
    w = np.asarray(w_uk, dtype=np.float64)
    if w.ndim == 2:
        w = w.reshape(w.shape[0], m, p)
    lat = w.shape[0]
    dev = device or torch.device("cuda", torch.cuda.current_device())
    latp = -(-lat // 8) * 8  # K1 streams weight rows in 16-byte vectors
    packed = np.zeros((m, p, latp))
    packed[:, :, :lat] = np.transpose(w, (1, 2, 0))
    qt = torch.as_tensor(q[None], dtype=torch.float32, device=dev).to(torch.bfloat16)
    qr = torch.zeros((1, m, 16), dtype=torch.bfloat16, device=dev)
    wt = torch.as_tensor(packed, dtype=torch.float32, device=dev).to(torch.bfloat16)
    q_abs, _ = ops.absorb_query(qt, qr, wt, 1, latp, 1.0)
    return q_abs[0, 0, :, :lat].double().cpu().numpy()


# ----------------------------------------------------------------------------- attention
def _queries_to_device(cfg: AttnConfig, layout: RowLayout, q_nope, q_rope, heads, device):
    qn = torch.as_tensor(np.asarray(q_nope)[list(heads)] if not torch.is_tensor(q_nope) else q_nope[list(heads)],
                         dtype=torch.float32, device=device)
    qr_src = torch.as_tensor(np.asarray(q_rope)[list(heads)] if not torch.is_tensor(q_rope) else q_rope[list(heads)],
                             dtype=torch.float32, device=device)
    qr = torch.zeros((len(heads), layout.drp), dtype=torch.float32, device=device)
    qr[:, :layout.dr] = qr_src
    return qn.to(torch.bfloat16)[None].contiguous(), qr.to(torch.bfloat16)[None].contiguous()


def _run_units(cfg: AttnConfig, cache: PagedLatentCache, lw: LocalWeights, qn, qr, upproj: int, alpha: float):
    layout = cache.layout
    dev = cache.paged.device
    w_uk, w_uv = lw.packed(layout, dev)
    sub, dls = layout.geometry
    nb = layout.nb
    pc = cache.paged
    nsplit = ops.default_splits(1, max(cache.n, 1), nb, sub)
    q_abs, q_rs = ops.absorb_query(qn, qr, w_uk, nb, layout.dlp, ops.score_scale(cfg.tau))
    o_part, lse = ops.decode_partials(q_abs, q_rs, pc.pool, pc.block_table, pc.seqlens, pc.page_size, nb, sub, dls,
                                      nsplit)
    return ops.combine(o_part, lse, w_uv, alpha, per_branch=(upproj == 2))


def attend_local(cfg: AttnConfig, local_w, own: Ownership, cache: PagedLatentCache, queries: dict) -> list:
    """Per-head contributions of one computing unit for the newest token (decode.py:204-230).

    One contribution per (head, unit), in unit order, like the reference. Charges the
    cache's read counter with every element a real device reads: each owned stream once.
    """
    _check_served(cfg)
    if not isinstance(cache, PagedLatentCache):
        raise RoutingError("attend_local on the B200 path needs a PagedLatentCache (new_cache)")
    if cfg.variant == "gqa":
        from .gqa import attend_local_gqa

        return attend_local_gqa(cfg, own, cache, queries)
    if cache.n == 0:
        raise ConfigError("cache read: stream 'rope' is empty")
    heads = list(own.units[0].heads)
    if any(list(u.heads) != heads for u in own.units):
        raise ConfigError("B200 path: all units of one owner must serve the same heads")
    if not isinstance(local_w, LocalWeights):
        lw = LocalWeights(local_w)
    else:
        lw = local_w
    qn, qr = _queries_to_device(cfg, cache.layout, queries["q_nope"], queries["q_rope"], heads, cache.paged.device)
    per_unit = _run_units(cfg, cache, lw, qn, qr, upproj=2, alpha=1.0)[0].double().cpu().numpy()
    cache.reads += cache.n * cache.row_elements()
    contribs = []
    for i, _unit in enumerate(own.units):
        contribs.extend((head, per_unit[i, j]) for j, head in enumerate(heads))
    return contribs


def reduce_contributions(cfg: AttnConfig, contribs: list) -> tuple[np.ndarray, str]:  # decode.py:264-285
    out = np.zeros((cfg.h, cfg.head_out_dim))
    counts = np.zeros(cfg.h, dtype=int)
    for head, vec in contribs:
        out[head] += vec
        counts[head] += 1
    if (counts == 0).any():
        missing = np.nonzero(counts == 0)[0].tolist()
        raise IntegrityError(f"no contribution for heads {missing}")
    kind = "concat" if (counts == 1).all() else "sum"
    if cfg.variant == "mlra":
        out *= calib_factors(cfg).alpha_attn
    return out, kind


# ----------------------------------------------------------------------------- decode steps
class _StepState:
    """Per-(config, weights) device state for the single-sequence drop-in step."""

    def __init__(self, cfg: AttnConfig, w, device):
        if cfg.variant == "gqa":
            from .projections import GqaProjector

            self.projector = GqaProjector(cfg, w, device)
        else:
            self.projector = LatentProjector(cfg, w, device)
        self.own = full_ownership(cfg)
        self.lw = local_weights(cfg, w, self.own)


_STATE: dict = {}


def _state(cfg: AttnConfig, w, device) -> _StepState:
    key = (cfg, id(w), str(device))
    st = _STATE.get(key)
    if st is None or st.__dict__.get("_w") is not w:
        st = _StepState(cfg, w, device)
        st._w = w
        _STATE[key] = st
    return st


def _owned_blocks(cfg: AttnConfig, layout: RowLayout) -> tuple[int, int, int]:
    """(branches, first block, block count) of a latent layout's units, for the fused K0."""
    if cfg.variant == "mla":
        return 1, 0, 1
    blocks = [int(u.rsplit("_b", 1)[1]) for u in layout.units]
    if blocks != list(range(blocks[0], blocks[0] + len(blocks))):
        raise ConfigError(f"owned latent blocks {blocks} are not contiguous")
    return 4, blocks[0], len(blocks)


def append_token_latent(cfg: AttnConfig, st: "_StepState", cache: PagedLatentCache, hidden: torch.Tensor,
                        pos: int) -> None:
    """Write side of one decode step for a latent-family cache: the raw down-projections
    (h W^DKV, h W^KR -- pre-attention GEMVs, torch) then the fused K0 kernel (rmsnorm*alpha_kv,
    owned blocks, rope, padding, paged append)."""
    branches, block0, nblocks = _owned_blocks(cfg, cache.layout)
    proj = st.projector
    cache.append_latent(hidden @ proj.w_dkv, hidden @ proj.w_kr, pos, branches=branches, block0=block0,
                        nblocks=nblocks, alpha_kv=proj.alpha_kv)


def absorbed_decode_step(cfg: AttnConfig, w, cache: PagedLatentCache, h_t) -> tuple[np.ndarray, PagedLatentCache]:
    """Cache-append plus one attention step without per-head KV expansion (decode.py:290-306)."""
    _check_served(cfg)
    dev = cache.paged.device
    st = _state(cfg, w, dev)
    pos = cache.pos_offset + cache.n
    if cfg.variant == "gqa":
        # zoo projections (zoo.py:47-58): append k, v rows, attend on the cached heads
        hidden = torch.as_tensor(np.asarray(h_t, dtype=np.float64).reshape(1, cfg.d), dtype=torch.float32, device=dev)
        q, k, v = st.projector(hidden, torch.tensor([pos], device=dev))
        cache.append_packed(cache.layout.pack_rows({"k": k[0], "v": v[0]}, device=dev)[None])
        contribs = attend_local(cfg, {}, st.own, cache, {"q": q[0]})
        out, _ = reduce_contributions(cfg, contribs)
        return out, cache
    hidden = torch.as_tensor(np.asarray(h_t, dtype=np.float64).reshape(1, cfg.d), dtype=torch.float32, device=dev)
    append_token_latent(cfg, st, cache, hidden, pos)
    q_nope, q_rope = st.projector.queries(hidden, torch.tensor([pos], device=dev))
    qn, qr = _queries_to_device(cfg, cache.layout, q_nope[0], q_rope[0], list(range(cfg.h)), dev)
    alpha = calib_factors(cfg).alpha_attn if cfg.variant == "mlra" else 1.0
    out = _run_units(cfg, cache, st.lw, qn, qr, upproj=1, alpha=alpha)
    cache.reads += cache.n * cache.row_elements()
    return out[0].double().cpu().numpy(), cache


def decode_step(cfg: AttnConfig, w, cache, h_t, mode: str = "absorbed"):  # decode.py:341-348
    if mode == "absorbed":
        return absorbed_decode_step(cfg, w, cache, h_t)
    if mode == "naive":
        raise RoutingError("naive decode (per-head K/V materialisation) is the CPU oracle's job; "
                           "the B200 path implements the absorbed form only")
    raise RoutingError(f"unknown decode mode {mode!r}")


# ----------------------------------------------------------------------------- batched engine
class DecodeEngine:
    """Batched decode attention for one device: B sequences in one paged pool.

    ``own`` selects what this device holds (full ownership = TP1; a tensor-parallel shard
    from ``tp.shard_ownership`` otherwise). ``decode_attention`` is the measured hot path:
    K1 (absorb) -> K2 (split-KV flash decode) -> K3 (merge, W^UV, branch sum, alpha).
    """

    def __init__(self, cfg: AttnConfig, w, own: Ownership | None = None, *, batch: int, max_tokens: int,
                 page_size: int = 128, device=None, nsplit: int | None = None, page_order=None,
                 alpha: float | None = None):
        _check_served(cfg)
        if cfg.variant == "gqa":
            raise RoutingError("DecodeEngine serves the latent family; use gqa.GqaDecodeEngine for gqa")
        self.cfg = cfg
        self.own = own or full_ownership(cfg)
        self.layout = row_layout(cfg, self.own)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.heads = list(self.own.units[0].heads)
        self.cache = PagedCache(self.layout, batch, max_tokens, page_size, self.device, page_order)
        lw = local_weights(cfg, w, self.own)
        self.w_uk, self.w_uv = lw.packed(self.layout, self.device)
        self.sub, self.dls = self.layout.geometry
        self.scale = ops.score_scale(cfg.tau)
        if alpha is None:
            alpha = calib_factors(cfg).alpha_attn if cfg.variant == "mlra" else 1.0
        self.alpha = float(alpha)
        self.nsplit = nsplit or ops.default_splits(batch, max_tokens, self.layout.nb, self.sub)
        hl = len(self.heads)
        self.workspace = ops.DecodeWorkspace(batch, hl, self.layout.nb, self.layout.dlp, self.layout.drp, self.nsplit,
                                             self.device)
        self.out = torch.empty((batch, hl, cfg.d_h), dtype=torch.float32, device=self.device)

    @property
    def batch(self) -> int:
        return self.cache.batch

    def prepare_queries(self, q_nope, q_rope) -> tuple[torch.Tensor, torch.Tensor]:
        """[B, h, d_h] / [B, h, dr] (any float, host or device) -> this device's heads, bf16, padded rope."""
        qn = torch.as_tensor(q_nope, device=self.device)[:, self.heads].to(torch.bfloat16).contiguous()
        qr_src = torch.as_tensor(q_rope, device=self.device)[:, self.heads]
        qr = torch.zeros((qr_src.shape[0], len(self.heads), self.layout.drp), dtype=torch.bfloat16, device=self.device)
        qr[..., :self.layout.dr] = qr_src.to(torch.bfloat16)
        return qn, qr

    def decode_attention(self, q_nope: torch.Tensor, q_rope: torch.Tensor, out: torch.Tensor | None = None):
        """One decode-attention step over the cache: bf16 [B, h_local, d_h] / [B, h_local, drp]
        queries on this device -> fp32 [B, h_local, d_h] (alpha-scaled, branch-summed)."""
        c = self.cache
        return ops.decode_step(q_nope, q_rope, self.w_uk, self.w_uv, c.pool, c.block_table, c.seqlens, c.page_size,
                               self.layout.nb, self.sub, self.dls, self.nsplit, self.scale, self.alpha,
                               self.workspace, out=self.out if out is None else out)
