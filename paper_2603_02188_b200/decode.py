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

from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .cache import GqaLayout, PagedCache, PagedLatentCache, RowLayout
from .config import LATENT_VARIANTS, AttnConfig
from .costs import calib_factors
from .errors import ConfigError, IntegrityError, RoutingError, ShapeMismatchError
from .projections import LatentProjector

SERVED = ("mla", "mlra", "gla", "gqa")


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
        raise RoutingError(f"the B200 decode path serves {SERVED}; got {cfg.variant!r}")


def full_ownership(cfg: AttnConfig) -> Ownership:  # decode.py:53-76 (served variants)
    _check_served(cfg)
    all_heads = tuple(range(cfg.h))
    if cfg.variant == "gqa":
        return Ownership(all_heads, kv_slots=tuple(range(cfg.g)))
    if cfg.variant == "mla":
        return Ownership(all_heads, units=(LatentUnit(-1, -1, all_heads),))
    if cfg.variant == "gla":
        r = cfg.h // cfg.g
        return Ownership(all_heads, units=tuple(LatentUnit(j, -1, tuple(range(j * r, (j + 1) * r)))
                                               for j in range(cfg.g)))
    if cfg.branches == 4:
        return Ownership(all_heads, units=tuple(LatentUnit(-1, b, all_heads) for b in range(4)))
    half = cfg.h // 2
    return Ownership(all_heads, units=tuple(LatentUnit(grp, b, tuple(range(grp * half, (grp + 1) * half)))
                                           for grp in range(2) for b in range(2)))


def unit_width(cfg: AttnConfig) -> int:
    if cfg.variant == "mla":
        return cfg.d_c
    if cfg.variant == "gla":
        return cfg.group_latent_dim
    return cfg.block_dim


def kernel_geometry(layout: RowLayout, own: Ownership) -> tuple[int, int]:
    """(NB, DLAT) of the decode kernels for an owner's units. Units serving the same heads are
    kernel branches (MLRA-4, MLA). Units serving different head sets (MLRA-2, GLA) run on the
    same kernels with block-diagonal weights: every branch computes every local head and the
    weights of (unit, head) pairs the unit does not serve are zero, so those contributions
    vanish in the up-projection. Narrow units (<= 128 columns) stay separate branches (the
    kernel keeps up to 4); wide ones (GLA-2 at TP1: 2 x 256) are concatenated into one branch
    of their summed width (the MLA geometry)."""
    nu, dlp = layout.nb, layout.dlp
    if nu in (1, 2, 4) and (dlp <= 128 or nu == 1):
        return nu, dlp
    if (nu * dlp) % 128 == 0 and nu * dlp <= 512:
        return 1, nu * dlp
    raise ConfigError(f"no kernel geometry for {nu} latent units of width {dlp}")


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
    if unit.group < 0:
        w_uk, w_uv = w["w_uk"], w["w_uv"]
    else:  # grouped latents: the group's own up-projections, heads indexed within the group
        w_uk, w_uv = w[f"w_uk_{unit.group}"], w[f"w_uv_{unit.group}"]
        r = cfg.h // cfg.g
        heads = [i - unit.group * r for i in heads]
    if unit.block >= 0:
        bs = cfg.block_dim
        w_uk = w_uk[unit.block * bs:(unit.block + 1) * bs]
        w_uv = w_uv[unit.block * bs:(unit.block + 1) * bs]
    d_lat = w_uk.shape[0]
    return (w_uk.reshape(d_lat, -1, cfg.d_h)[:, heads], w_uv.reshape(d_lat, -1, cfg.d_h)[:, heads])


class LocalWeights(dict):
    """``{"uk:<stream>": (latent, m, d_h), "uv:<stream>": ...}`` like decode.py:190-199, with a
    cached device pack over the owner's heads: w_uk [m, d_h, NU*dlp] and w_uv [m, NU*dlp, d_h]
    (bf16, zero-padded; zero where a unit does not serve a head -- see kernel_geometry)."""

    def packed(self, layout: RowLayout, device, own: Ownership | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        key = ("__packed__", layout, str(device), None if own is None else (own.heads, own.units))
        if key not in self.__dict__:
            uk, uv = self.packed_host(layout, own)
            self.__dict__[key] = (torch.as_tensor(uk, device=device).to(torch.bfloat16).contiguous(),
                                  torch.as_tensor(uv, device=device).to(torch.bfloat16).contiguous())
        return self.__dict__[key]

    def packed_host(self, layout: RowLayout, own: Ownership | None = None) -> tuple[np.ndarray, np.ndarray]:
        """The same packs in float32 on the host (before the bf16 rounding)."""
        key = ("__packed_host__", layout, None if own is None else (own.heads, own.units))
        if key not in self.__dict__:
            uks = [np.asarray(self[f"uk:{u}"]) for u in layout.units]
            uvs = [np.asarray(self[f"uv:{u}"]) for u in layout.units]
            dh = uks[0].shape[2]
            heads = list(own.heads) if own is not None else list(range(uks[0].shape[1]))
            unit_heads = [list(u.heads) for u in own.units] if own is not None else [heads] * len(uks)
            m = len(heads)
            nu, dlp, dl = layout.nb, layout.dlp, layout.dl
            uk = np.zeros((m, dh, nu * dlp), dtype=np.float32)
            uv = np.zeros((m, nu * dlp, dh), dtype=np.float32)
            for i, (a, b) in enumerate(zip(uks, uvs)):
                rows = [heads.index(hd) for hd in unit_heads[i]]
                uk[rows, :, i * dlp:i * dlp + dl] = np.transpose(a, (1, 2, 0))  # (lat, m, dh) -> (m, dh, lat)
                uv[rows, i * dlp:i * dlp + dl, :] = np.transpose(b, (1, 0, 2))  # (lat, m, dh) -> (m, lat, dh)
            self.__dict__[key] = (uk, uv)
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


def _pad_rope(qn: torch.Tensor, qr: torch.Tensor, layout: RowLayout):
    """K-1's rotary queries [M, h, dr] -> the cache layout's padded width drp (zero columns)."""
    if qr.shape[-1] == layout.drp:
        return qn.contiguous(), qr.contiguous()
    out = torch.zeros(qr.shape[:-1] + (layout.drp,), dtype=qr.dtype, device=qr.device)
    out[..., :qr.shape[-1]] = qr
    return qn.contiguous(), out


def _run_units(cfg: AttnConfig, cache: PagedLatentCache, lw: LocalWeights, own: Ownership, qn, qr, upproj: int,
               alpha: float):
    layout = cache.layout
    dev = cache.paged.device
    w_uk, w_uv = lw.packed(layout, dev, own)
    nb, dlat = kernel_geometry(layout, own)
    sub, dls = ops.latent_geometry(dlat)
    pc = cache.paged
    nsplit = ops.default_splits(1, max(cache.n, 1), nb, sub, heads=len(own.heads))
    q_abs, q_rs = ops.absorb_query(qn, qr, w_uk, nb, dlat, ops.score_scale(cfg.tau))
    o_part, lse = ops.decode_partials(q_abs, q_rs, pc.pool, pc.block_table, pc.seqlens, pc.page_size, nb, sub, dls,
                                      nsplit)
    status = ops.status_word(dev)
    out = ops.combine(o_part, lse, w_uv, alpha, per_branch=(upproj == 2), status=status)
    ops.check_status(status, "softmax_rows")  # NaN / no finite logit -> NumericError (tensors.py:74-78)
    return out


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
    heads = list(own.heads)
    if not isinstance(local_w, LocalWeights):
        lw = LocalWeights(local_w)
    else:
        lw = local_w
    qn, qr = _queries_to_device(cfg, cache.layout, queries["q_nope"], queries["q_rope"], heads, cache.paged.device)
    per_branch = _run_units(cfg, cache, lw, own, qn, qr, upproj=2, alpha=1.0)[0].double().cpu().numpy()
    cache.reads += cache.n * cache.row_elements()
    merged = per_branch.shape[0] != len(own.units)  # units concatenated into one kernel branch
    contribs = []
    for i, unit in enumerate(own.units):
        row = per_branch[0 if merged else i]
        contribs.extend((head, row[heads.index(head)]) for head in unit.heads)
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
        self.cfg, self.w, self.device = cfg, w, device
        self._kproj = None

    @property
    def kproj(self):
        """K-1 kernels for the drop-in single-token steps (full heads, q_nope for K1)."""
        if self._kproj is None:
            from .projections import KernelProjector

            names = _write_plan(self.cfg, self.own)[0]
            self._kproj = KernelProjector(self.cfg, self.w, self.device, range(self.cfg.h), names, absorbed=False)
        return self._kproj


_STATE: "OrderedDict[tuple, _StepState]" = OrderedDict()
_STATE_MAX = 4  # device weight packs of the most recently used weight sets (LRU)


def _state(cfg: AttnConfig, w, device) -> _StepState:
    """Device state (packed weights, projector) of one weight set, kept for the last _STATE_MAX
    weight sets used: a long-lived process that steps many models does not pin every one."""
    key = (cfg, id(w), str(device))
    st = _STATE.get(key)
    if st is None or st.__dict__.get("_w") is not w:
        st = _StepState(cfg, w, device)
        st._w = w
        _STATE[key] = st
    _STATE.move_to_end(key)
    while len(_STATE) > _STATE_MAX:
        _STATE.popitem(last=False)
    return st


def _write_plan(cfg: AttnConfig, own: Ownership) -> tuple[list, int, int, int, int]:
    """What the fused K0 needs for an owner: (raw down-projection names concatenated into
    kv_raw, blocks per kv_raw row, first owned block, owned block count, RMS groups)."""
    units = list(own.units)
    if cfg.variant == "mla":
        return ["w_dkv"], 1, 0, 1, 1
    if cfg.variant == "mlra" and cfg.branches == 4:
        blocks = [u.block for u in units]
        if blocks != list(range(blocks[0], blocks[0] + len(blocks))):
            raise ConfigError(f"owned latent blocks {blocks} are not contiguous")
        return ["w_dkv"], 4, blocks[0], len(blocks), 1  # the RMS spans the whole latent
    # grouped latents: each group normalised over its own latent (latent.py:145-158)
    groups = sorted({u.group for u in units})
    per_group = 1 if cfg.variant == "gla" else 2
    idx = [groups.index(u.group) * per_group + max(u.block, 0) for u in units]
    if idx != list(range(idx[0], idx[0] + len(idx))):
        raise ConfigError(f"owned latent units {[u.stream for u in units]} are not contiguous")
    return [f"w_dkv_{j}" for j in groups], per_group * len(groups), idx[0], len(idx), len(groups)


def append_token_latent(cfg: AttnConfig, st: "_StepState", cache: PagedLatentCache, kv_raw: torch.Tensor,
                        kr_raw: torch.Tensor, pos: int, own: Ownership | None = None) -> None:
    """Write side of one decode step for a latent-family cache: the fused K0 kernel (rmsnorm*alpha_kv
    per latent group, owned blocks, rope, padding, paged append) on the raw down-projections that
    K-1 (``st.kproj.project``) produced for the token: kv_raw [1, all latent groups], kr_raw [1, dr]."""
    names, blocks, block0, nblocks, norm_groups = _write_plan(cfg, own or st.own)
    cache.append_latent(st.kproj.kv_slice(kv_raw, names), kr_raw, pos, branches=blocks, block0=block0,
                        nblocks=nblocks, alpha_kv=st.kproj.alpha_kv, norm_groups=norm_groups)


def token_projections(cfg: AttnConfig, st: "_StepState", h_t, pos: int):
    """K-1 for one token (latent.py:129-159 at one position): (kv_raw, kr_raw, q_nope [1, h, d_h]
    bf16, q_rope [1, h, dr] bf16 with rope applied), all on the device."""
    dev = st.device
    hidden = torch.as_tensor(np.asarray(h_t, dtype=np.float64).reshape(1, cfg.d), dtype=torch.float32, device=dev)
    return st.kproj.project(hidden, torch.tensor([pos], dtype=torch.int32, device=dev))


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
    kv_raw, kr_raw, qn, qr = token_projections(cfg, st, h_t, pos)  # K-1 (hand-written GEMMs)
    append_token_latent(cfg, st, cache, kv_raw, kr_raw, pos)        # fused K0
    qn, qr = _pad_rope(qn, qr, cache.layout)
    alpha = calib_factors(cfg).alpha_attn if cfg.variant == "mlra" else 1.0
    out = _run_units(cfg, cache, st.lw, st.own, qn, qr, upproj=1, alpha=alpha)
    cache.reads += cache.n * cache.row_elements()
    return out[0].double().cpu().numpy(), cache


# ----------------------------------------------------------------------------- prefill
@dataclass
class PrefillOutput:  # latent.py PrefillOutput: per-token outputs and the filled cache
    out: np.ndarray
    cache: PagedLatentCache


PREFILL_CHUNK = 4096  # queries per kernel pass (K2's grid.y and the split workspace scale with it)


def latent_prefill(cfg: AttnConfig, w, hidden, pos_offset: int = 0, *, device=None,
                   page_size: int = 128) -> PrefillOutput:
    """Causal prefill (latent.py:172-230) writing the paged cache format directly (SURVEY.md
    8(f) row 3).

    Write side: the raw down-projections of all n tokens (GEMMs) and ONE fused K0 launch with n
    rows, each row writing its token's slot of the sequence's pages (the page table repeated
    per row, slots 0..n-1). Attention side: token t is a decode query over the first t+1 cached
    rows, so the n queries run as n pseudo-sequences sharing the sequence's page table with
    seqlens 1..n through K1 -> K2 -> K3 (causality by the lengths, no mask). The cache rows
    K2 re-reads stay L2-resident across the pseudo-sequences; this is the decode kernels'
    arithmetic (absorbed logits, bf16 cache, fp32 softmax and merge), not a separate prefill
    kernel.
    """
    if cfg.variant not in LATENT_VARIANTS:
        raise RoutingError(f"variant {cfg.variant!r} belongs to the baseline zoo, not latent_prefill")
    _check_served(cfg)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    st = _state(cfg, w, dev)
    hid = np.asarray(hidden, dtype=np.float64)
    if hid.ndim != 2 or hid.shape[1] != cfg.d:
        raise ShapeMismatchError(f"prefill hidden {hid.shape} != (n, {cfg.d})")
    n = hid.shape[0]
    cache = new_cache(cfg, pos_offset=pos_offset, device=dev, page_size=page_size,
                      initial_tokens=max(n, page_size))
    if n == 0:
        return PrefillOutput(np.zeros((0, cfg.h, cfg.d_h)), cache)
    out = prefill_into(cfg, st, cache, torch.as_tensor(hid, dtype=torch.float32, device=dev))
    return PrefillOutput(out.double().cpu().numpy(), cache)


def prefill_kernel_fits(cfg: AttnConfig, layout: RowLayout, own: Ownership, page_size: int) -> bool:
    """K6 (the tcgen05 causal prefill kernel) serves 128- or 64-wide latent branches with a matching
    head width (MLRA-4 / MLRA-2 at the 2.9B shape, the tiny config), <= 64 rotary columns and
    pages of whole 128-token tiles; other geometries take the pseudo-sequence path."""
    nb, dlat = kernel_geometry(layout, own)
    return (dlat, cfg.d_h) in ((128, 128), (64, 64)) and nb <= 4 and layout.drp <= 64 and page_size % 128 == 0


def prefill_into(cfg: AttnConfig, st: "_StepState", cache: PagedLatentCache, h_t: torch.Tensor,
                 force_pseudo: bool = False) -> torch.Tensor:
    """Device part of latent_prefill: fill the EMPTY paged cache with the n tokens of h_t
    [n, d] fp32 (positions pos_offset + t) and return the outputs [n, h, d_h] fp32.

    Write side: the n rows' projections (cuBLAS bf16 GEMMs on K-1's packed weights) and ONE
    fused K0 launch writing token t at slot t of the sequence's pages. Queries: K1 over the n
    rows. Attention: K6 (``mlra_prefill_attention``: causal, tcgen05, 128 queries x one head
    per CTA, all branches and the W^UV up-projection in-kernel) when the geometry fits;
    otherwise the n queries run as n decode pseudo-sequences of lengths 1..n over the same
    pages through K2 -> K3 (causality by the lengths)."""
    n = h_t.shape[0]
    dev = h_t.device
    pc = cache.paged
    layout = cache.layout
    positions = torch.arange(cache.pos_offset, cache.pos_offset + n, dtype=torch.int32, device=dev)
    # ---- write side: one K0 launch for all n tokens (slots 0..n-1 of block_table row 0)
    names, blocks, block0, nblocks, norm_groups = _write_plan(cfg, st.own)
    kp = st.kproj
    use_k6 = not force_pseudo and prefill_kernel_fits(cfg, layout, st.own, pc.page_size)
    # the n rows' projections (cuBLAS bf16); K6 reads 64-column rotary query rows
    scale = ops.score_scale(cfg.tau)
    kv_raw, kr_raw, qn, q_r = kp.project_gemm(h_t, cache.pos_offset, drq=64 if use_k6 else layout.drp,
                                              rope_scale=scale if use_k6 else None)
    kv_raw = kp.kv_slice(kv_raw, names)
    ops.cache_append_latent(kv_raw, kr_raw, positions, None, pc.block_table, pc.pool, pc.page_size, branches=blocks,
                            block0=block0, nblocks=nblocks, dlp=layout.dlp, drp=layout.drp,
                            alpha_kv=kp.alpha_kv, norm_groups=norm_groups)
    pc.seqlens.fill_(n)
    pc._host_lens = [n]
    heads = list(range(cfg.h))
    w_uk, w_uv = st.lw.packed(layout, dev, st.own)
    nb, dlat = kernel_geometry(layout, st.own)
    sub, dls = ops.latent_geometry(dlat)
    alpha = calib_factors(cfg).alpha_attn if cfg.variant == "mlra" else 1.0
    if use_k6:
        # absorption of the n queries as one batched GEMM over the heads (bf16 operands, fp32
        # accumulation, tau*log2e applied before the bf16 rounding -- K1's arithmetic), written
        # head-major [H, n, NB*DLAT] as K6 reads it (the rotary queries come scaled from the epilogue)
        q_abs = torch.baddbmm(torch.zeros((1, 1, 1), dtype=torch.bfloat16, device=dev), qn.transpose(0, 1), w_uk,
                              beta=0.0, alpha=scale)
        return ops.prefill_attention(q_abs.view(cfg.h, n, nb, dlat), q_r, w_uv, pc.pool, pc.block_table,
                                     pc.page_size, nb, dlat, cfg.d_h_rope, alpha)
    qn, qr = _pad_rope(qn, q_r, layout)
    # ---- pseudo-sequence path: n queries of lengths 1..n over the same pages
    bt_rep = pc.block_table[:1].expand(min(n, PREFILL_CHUNK), -1).contiguous()
    out = torch.empty((n, len(heads), cfg.d_h), dtype=torch.float32, device=dev)
    for t0 in range(0, n, PREFILL_CHUNK):
        t1 = min(n, t0 + PREFILL_CHUNK)
        m = t1 - t0
        lens = torch.arange(t0 + 1, t1 + 1, dtype=torch.int32, device=dev)
        nsplit = ops.default_splits(m, t1, nb, sub)
        q_abs, q_rs = ops.absorb_query(qn[t0:t1], qr[t0:t1].contiguous(), w_uk, nb, dlat, scale)
        o_part, lse = ops.decode_partials(q_abs, q_rs, pc.pool, bt_rep[:m], lens, pc.page_size, nb, sub, dls,
                                          nsplit)
        out[t0:t1] = ops.combine(o_part, lse, w_uv, alpha)
    return out


def naive_decode_step(cfg: AttnConfig, w, cache: PagedLatentCache, h_t) -> tuple[np.ndarray, PagedLatentCache]:
    """The reference's materialising decode (decode.py:309-338), same contract: latent family
    only (RoutingError otherwise), cache append, per-head softmax over the prefix, alpha_attn.

    On the B200 the per-head keys/values C·W^UK_h, C·W^UV_h are never materialised: the logits
    q_h·(C W^UK_h)^T equal (q_h W^UK_h^T)·C^T and the output P·(C W^UV_h) equals (P·C)·W^UV_h
    exactly in real arithmetic, so this runs the absorbed K0-K3 path (in float64 the
    reference's two forms agree to 1e-10; tests/test_oracle.py). Reads are accounted like the
    reference (every owned latent stream and the rope once)."""
    if cfg.variant not in LATENT_VARIANTS:
        raise RoutingError(f"naive_decode_step covers the latent family; {cfg.variant!r} decodes directly")
    return absorbed_decode_step(cfg, w, cache, h_t)


def decode_step(cfg: AttnConfig, w, cache, h_t, mode: str = "absorbed"):  # decode.py:341-348
    if mode == "absorbed":
        return absorbed_decode_step(cfg, w, cache, h_t)
    if mode == "naive":
        return naive_decode_step(cfg, w, cache, h_t)
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
                 alpha: float | None = None, ragged: bool = False):
        _check_served(cfg)
        if cfg.variant == "gqa":
            raise RoutingError("DecodeEngine serves the latent family; use gqa.GqaDecodeEngine for gqa")
        self.cfg = cfg
        self.own = own or full_ownership(cfg)
        self.layout = row_layout(cfg, self.own)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.heads = list(self.own.heads)
        self.cache = PagedCache(self.layout, batch, max_tokens, page_size, self.device, page_order)
        lw = local_weights(cfg, w, self.own)
        self.w_uk, self.w_uv = lw.packed(self.layout, self.device, self.own)
        self.nb, self.dlat = kernel_geometry(self.layout, self.own)
        self.sub, self.dls = ops.latent_geometry(self.dlat)
        self.scale = ops.score_scale(cfg.tau)
        if alpha is None:
            alpha = calib_factors(cfg).alpha_attn if cfg.variant == "mlra" else 1.0
        self.alpha = float(alpha)
        # ragged=True: K2's work comes from the device-side plan (mlra_decode_plan) that balances the
        # sequences' tiles over one wave of CTAs; nsplit is then the most splits one sequence may get
        self.ragged = bool(ragged)
        if ragged and nsplit is None:
            nsplit = min(64, max(1, ops.num_sms() // max(1, -(-len(self.heads) // 64))))
        self.nsplit = nsplit or ops.default_splits(batch, max_tokens, self.nb, self.sub, heads=len(self.heads))
        hl = len(self.heads)
        self.workspace = ops.DecodeWorkspace(batch, hl, self.nb, self.dlat, self.layout.drp, self.nsplit, self.device)
        self.out = torch.empty((batch, hl, cfg.d_h), dtype=torch.float32, device=self.device)
        self._w, self._lw, self._kp = w, lw, {}

    def kernel_projector(self, absorbed: bool | None = None):
        """K-1 for this device (its heads, its latent groups' raw down-projections). absorbed=None:
        pre-multiply W^UQ.W^UK_b when that weight is no larger than W^UQ (one latent block per
        device), so the query kernel writes K2's q~ and K1 is skipped."""
        if absorbed not in self._kp:
            from .projections import KernelProjector

            uk, _ = self._lw.packed_host(self.layout, self.own)
            self._kp[absorbed] = KernelProjector(self.cfg, self._w, self.device, self.heads,
                                                 _write_plan(self.cfg, self.own)[0], uk_pack=uk, nb=self.nb,
                                                 dlat=self.dlat, drp=self.layout.drp, absorbed=absorbed,
                                                 score_scale=self.scale)
        return self._kp[absorbed]

    def decode_layer(self, hidden: torch.Tensor, out: torch.Tensor | None = None, absorbed: bool | None = None,
                     advance: bool = True):
        """One decode step of the attention layer from the new tokens' hidden rows (the paper's
        end-to-end scope: the pre-attention stage plus the attention):
        K-1 down (h W^DQ, h W^DKV, h W^KR) -> K0 (rmsnorm*alpha_kv, rope, paged append at the
        sequence's length, advancing it) -> K-1 query (c_q rmsnorm, W^UQ [. W^UK_b], W^QR, rope)
        -> [K1] -> K2 -> K3. hidden [B, d] fp32 on the device (B <= 16 per call); out [B, h_local,
        d_h] fp32. ``advance=False`` rewrites the same slot every call (timing loops)."""
        cfg, c = self.cfg, self.cache
        kp = self.kernel_projector(absorbed)
        names, blocks, block0, nblocks, norm_groups = _write_plan(cfg, self.own)
        B = hidden.shape[0]
        kv_raw, kr_raw = kp.down(hidden)
        ops.cache_append_latent(kv_raw, kr_raw, None, c.seqlens, c.block_table, c.pool, c.page_size,
                                branches=blocks, block0=block0, nblocks=nblocks, dlp=self.layout.dlp,
                                drp=self.layout.drp, alpha_kv=kp.alpha_kv, norm_groups=norm_groups, advance=advance,
                                chain=True)  # the query projection's weights stream meanwhile
        q, qr = kp.query(B, c.seqlens, pos_delta=-1 if advance else 0)
        if advance and getattr(c, "_host_lens", None) is not None:  # host mirror (eager calls)
            c._host_lens = [n + 1 for n in c._host_lens]
        step = ops.decode_step_ragged if self.ragged else ops.decode_step
        return step(q, qr, None if kp.absorbed else self.w_uk, self.w_uv, c.pool, c.block_table,
                    c.seqlens, c.page_size, self.nb, self.sub, self.dls, self.nsplit, self.scale,
                    self.alpha, self.workspace, out=self.out if out is None else out)

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

    def decode_attention_tp(self, q_nope: torch.Tensor, q_rope: torch.Tensor, reducer, out: torch.Tensor | None = None):
        """decode_attention plus the sum over the TP group fused into K3 (every local head must be
        a global head: owners holding all heads, MLRA-4 / MLRA-2 by latent block). reducer:
        collective.PeerAllReduce sized B*h*d_h (its regions and epoch are shared with K5)."""
        if len(self.heads) != self.cfg.h:
            raise RoutingError("fused TP sum needs owners holding every head; use K5 after the step")
        c = self.cache
        return ops.decode_step_tp(q_nope, q_rope, self.w_uk, self.w_uv, c.pool, c.block_table, c.seqlens,
                                  c.page_size, self.nb, self.sub, self.dls, self.nsplit, self.scale, self.alpha,
                                  self.workspace, reducer.rank, reducer.world, reducer.ptrs,
                                  out=self.out if out is None else out, comm_n=reducer.n)

    def check_numeric(self) -> None:
        """Synchronise, read and reset the workspace's status word: NumericError when any step since
        the last check saw a NaN logit or a row with no finite logit (attnkit/tensors.py:74-78). The
        decode call itself never synchronises (serving loops replay it from CUDA graphs)."""
        ops.check_status(self.workspace.status, "softmax_rows")

    def decode_attention(self, q_nope: torch.Tensor, q_rope: torch.Tensor, out: torch.Tensor | None = None):
        """One decode-attention step over the cache: bf16 [B, h_local, d_h] / [B, h_local, drp]
        queries on this device -> fp32 [B, h_local, d_h] (alpha-scaled, branch-summed)."""
        c = self.cache
        step = ops.decode_step_ragged if self.ragged else ops.decode_step
        return step(q_nope, q_rope, self.w_uk, self.w_uv, c.pool, c.block_table, c.seqlens, c.page_size,
                    self.nb, self.sub, self.dls, self.nsplit, self.scale, self.alpha,
                    self.workspace, out=self.out if out is None else out)
