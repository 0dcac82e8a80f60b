"""CPU restatement (float64 numpy) of the reference decode path -- TEST INFRASTRUCTURE ONLY.

This module is the parity oracle for the B200 kernels. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl reference``
arm may import it; the product package ``paper_2603_02188_b200`` never does.

It restates, function by function, the reference kit's decode path
(/root/reference/pkg/src/attnkit, cited as ``attnkit/<file>:<line>``) for the
variants the B200 path serves (mla, mlra-4, mlra-2, gla, gqa) and is pinned against golden
vectors generated from the reference itself (``oracle/gen_golden.py`` ->
``tests/golden/*.npz``; checked by ``tests/test_oracle.py``).

Data model: instead of the reference's per-token Python lists
(``KvCache``, attnkit/cache.py:24-84) a cache here is a dict of stacked
``(n, ...)`` float64 arrays plus an element-read counter with the same
semantics as ``KvCache.read`` (attnkit/cache.py:59-66).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

LATENT = ("mla", "gla", "mlra")
TP_DEGREES = (1, 2, 4, 8)


class OracleError(Exception):
    pass


# ----------------------------------------------------------------------------- config
@dataclass(frozen=True)
class Cfg:
    """Subset of attnkit AttnConfig (attnkit/config.py:23-124) used by the decode path."""

    variant: str
    h: int
    d: int
    d_h: int
    d_h_rope: int = -1
    d_c: int = -1
    d_cq: int = -1
    g: int = 1
    branches: int = 0
    scaling: bool = False
    gated: bool = False

    def __post_init__(self):
        if self.d_h_rope < 0:
            object.__setattr__(self, "d_h_rope", self.d_h // 2)
        if self.d_c < 0:
            object.__setattr__(self, "d_c", 4 * self.d_h)
        if self.d_cq < 0:
            object.__setattr__(self, "d_cq", 4 * self.d_h)
        if self.variant == "mlra":
            object.__setattr__(self, "g", 2 if self.branches == 2 else 1)

    @property
    def tau(self) -> float:  # attnkit/config.py:100-112
        if self.variant in LATENT:
            return (self.d_h + self.d_h_rope) ** -0.5
        return self.d_h ** -0.5

    @property
    def block_dim(self) -> int:  # attnkit/config.py:114-117
        return self.d_c // 4

    @property
    def group_latent_dim(self) -> int:  # attnkit/config.py:119-121
        return self.d_c // self.g

    @property
    def grouped(self) -> bool:  # attnkit/weights.py:104-105 (gla, or mlra with two branches)
        return self.variant == "gla" or (self.variant == "mlra" and self.branches == 2)


def cfg_from(obj) -> Cfg:
    """Build a Cfg from any object with AttnConfig-like attributes (duck-typed)."""
    return Cfg(obj.variant, obj.h, obj.d, obj.d_h, obj.d_h_rope, obj.d_c, obj.d_cq, obj.g, obj.branches,
               bool(obj.scaling), bool(getattr(obj, "gated", False)))


# ----------------------------------------------------------------------------- substrate
def philox_key(seed: int, path: tuple) -> int:  # attnkit/tensors.py:20-27
    hsh = hashlib.blake2b(digest_size=16)
    hsh.update(str(int(seed)).encode())
    for label in path:
        hsh.update(b"/")
        hsh.update(str(label).encode())
    return int.from_bytes(hsh.digest(), "little")


def normal(seed: int, path: tuple, shape, sigma: float = 1.0) -> np.ndarray:  # attnkit/tensors.py:30-49
    if sigma == 0.0:
        return np.zeros(shape)
    gen = np.random.Generator(np.random.Philox(key=philox_key(seed, path)))
    return sigma * gen.standard_normal(size=shape, dtype=np.float64)


def softmax_rows(m: np.ndarray) -> np.ndarray:  # attnkit/tensors.py:67-80
    m = np.asarray(m, dtype=np.float64)
    if np.isnan(m).any():
        raise OracleError("softmax_rows: NaN in input")
    peak = np.max(m, axis=-1, keepdims=True)
    if np.isneginf(peak).any():
        raise OracleError("softmax_rows: row with no finite entry")
    e = np.exp(m - peak)
    return e / np.sum(e, axis=-1, keepdims=True)


def rmsnorm(m: np.ndarray, eps: float = 1e-6) -> np.ndarray:  # attnkit/tensors.py:83-87
    ms = np.mean(m * m, axis=-1, keepdims=True)
    return m / np.sqrt(ms + eps)


def rope_rotate(x: np.ndarray, positions, base: float = 10000.0) -> np.ndarray:  # attnkit/rope.py:36-66
    x = np.asarray(x, dtype=np.float64)
    dim = x.shape[-1]
    freqs = float(base) ** (-2.0 * np.arange(dim // 2, dtype=np.float64) / dim)
    ang = np.multiply.outer(np.asarray(list(positions), dtype=np.float64), freqs)
    ang = ang.reshape((x.shape[0],) + (1,) * (x.ndim - 2) + (dim // 2,))
    cos, sin = np.cos(ang), np.sin(ang)
    even, odd = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = even * cos - odd * sin
    out[..., 1::2] = even * sin + odd * cos
    return out


def calib_alphas(cfg: Cfg) -> tuple[float, float, float]:  # attnkit/latent.py:41-69
    if not cfg.scaling or cfg.variant not in LATENT:
        return 1.0, 1.0, 1.0
    if cfg.variant == "mla":
        q2, kv2, a2 = Fraction(cfg.d, cfg.d_cq), Fraction(cfg.d, cfg.d_c), Fraction(1)
    elif cfg.variant == "gla":
        q2, kv2, a2 = Fraction(cfg.d, cfg.d_cq), Fraction(cfg.g * cfg.d, cfg.d_c), Fraction(1)
    else:
        q2, kv2, a2 = Fraction(cfg.d, cfg.d_cq), Fraction(4 * cfg.d, cfg.d_c), Fraction(1, cfg.branches)
    return float(q2) ** 0.5, float(kv2) ** 0.5, float(a2) ** 0.5


def weight_shapes(cfg: Cfg) -> dict:  # attnkit/weights.py:45-99 (latent family + gqa)
    h, d, d_h = cfg.h, cfg.d, cfg.d_h
    if cfg.variant == "gqa":
        s = {"w_q": (d, h * d_h), "w_k": (d, cfg.g * d_h), "w_v": (d, cfg.g * d_h)}
    elif cfg.variant in LATENT:
        s = {"w_dq": (d, cfg.d_cq), "w_uq": (cfg.d_cq, h * d_h), "w_qr": (cfg.d_cq, h * cfg.d_h_rope),
             "w_kr": (d, cfg.d_h_rope)}
        if cfg.grouped:  # weights.py:85-91: one latent (and up-projections) per group
            r, dg = h // cfg.g, cfg.group_latent_dim
            for j in range(cfg.g):
                s[f"w_dkv_{j}"] = (d, dg)
                s[f"w_uk_{j}"] = (dg, r * d_h)
                s[f"w_uv_{j}"] = (dg, r * d_h)
        else:
            s.update({"w_dkv": (d, cfg.d_c), "w_uk": (cfg.d_c, h * d_h), "w_uv": (cfg.d_c, h * d_h)})
    else:
        raise OracleError(f"oracle covers the latent family and gqa, not {cfg.variant}")
    if cfg.gated:  # weights.py:98-99
        s["w_g"] = (d, h * d_h)
    s["w_o"] = (h * d_h, d)
    return s


def build_weights(cfg: Cfg, sigma: float, seed: int, path: tuple) -> dict:  # attnkit/weights.py:107-113
    return {name: normal(seed, path + (name,), shape, sigma) for name, shape in weight_shapes(cfg).items()}


# ----------------------------------------------------------------------------- projections
def latent_projections(cfg: Cfg, w: dict, hidden: np.ndarray, positions):  # attnkit/latent.py:129-159
    n = hidden.shape[0]
    positions = list(positions)
    aq, akv, _ = calib_alphas(cfg)
    c_q = aq * rmsnorm(hidden @ w["w_dq"])
    q_nope = (c_q @ w["w_uq"]).reshape(n, cfg.h, cfg.d_h)
    q_rope = rope_rotate((c_q @ w["w_qr"]).reshape(n, cfg.h, cfg.d_h_rope), positions)
    k_rope = rope_rotate(hidden @ w["w_kr"], positions)
    bs = cfg.block_dim
    if cfg.variant == "mla":
        latents = {"latent": akv * rmsnorm(hidden @ w["w_dkv"])}
    elif cfg.variant == "gla":  # latent.py:145-147: one normalised latent per group
        latents = {f"latent_{j}": akv * rmsnorm(hidden @ w[f"w_dkv_{j}"]) for j in range(cfg.g)}
    elif cfg.branches == 4:
        c_kv = akv * rmsnorm(hidden @ w["w_dkv"])
        latents = {f"latent_b{b}": c_kv[:, b * bs:(b + 1) * bs] for b in range(4)}
    else:  # mlra-2, latent.py:154-158: two blocks within each of the two group latents
        latents = {}
        for grp in range(2):
            c_grp = akv * rmsnorm(hidden @ w[f"w_dkv_{grp}"])
            for b in range(2):
                latents[f"latent_{grp}_{b}"] = c_grp[:, b * bs:(b + 1) * bs]
    return q_nope, q_rope, k_rope, latents


def gqa_projections(cfg: Cfg, w: dict, hidden: np.ndarray, positions):  # attnkit/zoo.py:47-58
    n = hidden.shape[0]
    q = rope_rotate((hidden @ w["w_q"]).reshape(n, cfg.h, cfg.d_h), positions)
    k = rope_rotate((hidden @ w["w_k"]).reshape(n, cfg.g, cfg.d_h), positions)
    v = (hidden @ w["w_v"]).reshape(n, cfg.g, cfg.d_h)
    return q, k, v


# ----------------------------------------------------------------------------- cache
@dataclass
class Cache:
    """Stacked-array restatement of KvCache (attnkit/cache.py:24-84)."""

    streams: dict = field(default_factory=dict)
    reads: int = 0
    pos_offset: int = 0

    @property
    def n(self) -> int:
        return next(iter(self.streams.values())).shape[0] if self.streams else 0

    def append(self, rows: dict) -> None:  # cache.py:44-57
        for k, v in rows.items():
            v = np.asarray(v, dtype=np.float64)[None]
            self.streams[k] = v if k not in self.streams else np.concatenate([self.streams[k], v])

    def read(self, name: str) -> np.ndarray:  # cache.py:59-66
        if name not in self.streams or self.streams[name].shape[0] == 0:
            raise OracleError(f"cache read: stream {name!r} is empty")
        out = self.streams[name]
        self.reads += out.size
        return out


def latent_streams(cfg: Cfg, w: dict, hidden: np.ndarray, pos_offset: int = 0) -> dict:
    """All cache rows for a prefix (what latent_prefill caches, attnkit/latent.py:172-230)."""
    _, _, k_rope, latents = latent_projections(cfg, w, hidden, range(pos_offset, pos_offset + hidden.shape[0]))
    streams = dict(latents)
    streams["rope"] = k_rope
    return streams


# ----------------------------------------------------------------------------- decode
def absorb_query(q_nope: np.ndarray, w_uk: np.ndarray) -> np.ndarray:  # attnkit/decode.py:155-167
    m, p = q_nope.shape
    if w_uk.ndim == 2:
        w_uk = w_uk.reshape(w_uk.shape[0], m, p)
    return np.einsum("mp,cmp->mc", q_nope, w_uk)


def stream_name(group: int, block: int) -> str:  # attnkit/cache.py:147-155
    if group < 0 and block < 0:
        return "latent"
    if block < 0:
        return f"latent_{group}"
    if group < 0:
        return f"latent_b{block}"
    return f"latent_{group}_{block}"


def unit(group: int, block: int, heads) -> tuple:
    """A latent unit as (stream, group, block, heads) -- attnkit/decode.py:31-41."""
    return (stream_name(group, block), group, block, tuple(heads))


def units(cfg: Cfg, heads=None):
    """Latent units of full ownership -- attnkit/decode.py:53-76."""
    all_heads = tuple(range(cfg.h))
    if cfg.variant == "mla":
        return [unit(-1, -1, all_heads)]
    if cfg.variant == "gla":
        r = cfg.h // cfg.g
        return [unit(j, -1, range(j * r, (j + 1) * r)) for j in range(cfg.g)]
    if cfg.branches == 4:
        return [unit(-1, b, all_heads) for b in range(4)]
    half = cfg.h // 2
    return [unit(grp, b, range(grp * half, (grp + 1) * half)) for grp in range(2) for b in range(2)]


def unit_weights(cfg: Cfg, w: dict, group: int, block: int, heads) -> tuple:  # attnkit/decode.py:170-187
    heads = list(heads)
    if group < 0:
        w_uk, w_uv, local = w["w_uk"], w["w_uv"], heads
    else:
        r = cfg.h // cfg.g
        w_uk, w_uv = w[f"w_uk_{group}"], w[f"w_uv_{group}"]
        local = [i - group * r for i in heads]
    if block >= 0:
        bs = cfg.block_dim
        w_uk, w_uv = w_uk[block * bs:(block + 1) * bs], w_uv[block * bs:(block + 1) * bs]
    d_lat = w_uk.shape[0]
    return (w_uk.reshape(d_lat, -1, cfg.d_h)[:, local], w_uv.reshape(d_lat, -1, cfg.d_h)[:, local])


def attend_latent(cfg: Cfg, w: dict, cache: Cache, q_nope, q_rope, unit_list, q_operand_scale=None) -> list:
    """attend_local, latent branch (attnkit/decode.py:217-230).

    q_operand_scale (test emulation only, default off): when set to s, the absorbed query and
    the rotary query enter the logits as bf16(q * s) / s -- the bf16 operands the B200 K1 hands
    K2 (the score scale s = tau*log2(e) folded in before the bf16 rounding)."""
    rope_hist = cache.read("rope")
    contribs = []
    for stream, group, block, heads in unit_list:
        latent_hist = cache.read(stream)
        uk, uv = unit_weights(cfg, w, group, block, heads)
        hl = list(heads)
        q_tilde = absorb_query(q_nope[hl], uk)
        q_r = q_rope[hl]
        if q_operand_scale is not None:
            q_tilde = bf16_round(q_tilde * q_operand_scale) / q_operand_scale
            q_r = bf16_round(q_r * q_operand_scale) / q_operand_scale
        logits = cfg.tau * (q_tilde @ latent_hist.T + q_r @ rope_hist.T)
        probs = softmax_rows(logits)
        mixed = probs @ latent_hist
        out = np.einsum("mc,cmp->mp", mixed, uv)
        contribs.extend((head, out[j]) for j, head in enumerate(heads))
    return contribs


def attend_gqa(cfg: Cfg, cache: Cache, q: np.ndarray, heads, kv_slots) -> list:
    """attend_local, gqa branch (attnkit/decode.py:232-240, :258-261; kv_map zoo.py:35-38)."""
    keys, values = cache.read("k"), cache.read("v")
    reps = cfg.h // cfg.g
    local = {slot: i for i, slot in enumerate(kv_slots)}
    gather = [local[hh // reps] for hh in heads]
    k_sel, v_sel = keys[:, gather], values[:, gather]
    logits = cfg.tau * np.einsum("mk,nmk->mn", q[list(heads)], k_sel)
    probs = softmax_rows(logits)
    out = np.einsum("mn,nmv->mv", probs, v_sel)
    return [(hh, out[j]) for j, hh in enumerate(heads)]


def reduce_contributions(cfg: Cfg, contribs: list) -> tuple:  # attnkit/decode.py:264-285
    out = np.zeros((cfg.h, cfg.d_h))
    counts = np.zeros(cfg.h, dtype=int)
    for head, vec in contribs:
        out[head] += vec
        counts[head] += 1
    if (counts == 0).any():
        raise OracleError(f"no contribution for heads {np.nonzero(counts == 0)[0].tolist()}")
    kind = "concat" if (counts == 1).all() else "sum"
    if cfg.variant == "mlra":
        out *= calib_alphas(cfg)[2]
    return out, kind


def decode_attention(cfg: Cfg, w: dict, streams: dict, q_nope: np.ndarray, q_rope: np.ndarray,
                     q_operand_scale=None) -> np.ndarray:
    """Steps 1-3 of absorbed decoding for one sequence over a complete cache (no append):
    the quantity the B200 K1+K2+K3 path computes. streams: latent stream(s) + 'rope'.
    q_operand_scale: see attend_latent (bf16 query operands, test emulation)."""
    cache = Cache(dict(streams))
    out, _ = reduce_contributions(cfg, attend_latent(cfg, w, cache, q_nope, q_rope, units(cfg), q_operand_scale))
    return out


def absorbed_decode_step(cfg: Cfg, w: dict, cache: Cache, h_t: np.ndarray) -> np.ndarray:
    """attnkit/decode.py:290-306: append this token's rows, then attend over the prefix."""
    pos = cache.pos_offset + cache.n
    hidden = np.asarray(h_t, dtype=np.float64).reshape(1, cfg.d)
    if cfg.variant == "gqa":
        q, k, v = gqa_projections(cfg, w, hidden, [pos])
        cache.append({"k": k[0], "v": v[0]})
        out, _ = reduce_contributions(cfg, attend_gqa(cfg, cache, q[0], range(cfg.h), range(cfg.g)))
        return out
    q_nope, q_rope, k_rope, latents = latent_projections(cfg, w, hidden, [pos])
    rows = {k: v[0] for k, v in latents.items()}
    rows["rope"] = k_rope[0]
    cache.append(rows)
    out, _ = reduce_contributions(cfg, attend_latent(cfg, w, cache, q_nope[0], q_rope[0], units(cfg)))
    return out


def naive_decode_step(cfg: Cfg, w: dict, cache: Cache, h_t: np.ndarray) -> np.ndarray:
    """attnkit/decode.py:309-338: per-head K/V materialised from the latent (oracle's oracle)."""
    pos = cache.pos_offset + cache.n
    hidden = np.asarray(h_t, dtype=np.float64).reshape(1, cfg.d)
    q_nope, q_rope, k_rope, latents = latent_projections(cfg, w, hidden, [pos])
    rows = {k: v[0] for k, v in latents.items()}
    rows["rope"] = k_rope[0]
    cache.append(rows)
    rope_hist = cache.read("rope")
    out = np.zeros((cfg.h, cfg.d_h))
    for stream, group, block, heads in units(cfg):
        latent_hist = cache.read(stream)
        uk, uv = unit_weights(cfg, w, group, block, heads)
        for j, head in enumerate(heads):
            k_head = latent_hist @ uk[:, j]
            v_head = latent_hist @ uv[:, j]
            logits = cfg.tau * (q_nope[0][head] @ k_head.T + q_rope[0][head] @ rope_hist.T)
            out[head] += softmax_rows(logits[None])[0] @ v_head
    if cfg.variant == "mlra":
        out *= calib_alphas(cfg)[2]
    return out


# ----------------------------------------------------------------------------- tensor parallel
def _ranges(total: int, parts: int, axis: str) -> list:  # attnkit/tpsim.py:51-55
    if parts <= 0 or total % parts != 0:
        raise OracleError(f"cannot split {axis} of size {total} into {parts} shards")
    size = total // parts
    return [tuple(range(k * size, (k + 1) * size)) for k in range(parts)]


def shard_units(cfg: Cfg, phi: int, k: int):
    """(heads, units | kv_slots) of device k under phi-way TP (attnkit/tpsim.py:58-131)."""
    if phi not in TP_DEGREES:
        raise OracleError(f"unsupported TP degree {phi}")
    h = cfg.h
    all_heads = tuple(range(h))
    if cfg.variant == "gqa":
        g, r = cfg.g, h // cfg.g
        if phi <= g:
            slots = _ranges(g, phi, "KV-head axis")[k]
            return tuple(range(slots[0] * r, (slots[-1] + 1) * r)), slots
        per_group = phi // g
        if phi % g != 0 or r % per_group != 0:
            raise OracleError(f"gqa: cannot split {r} heads per KV head across {per_group} devices")
        group = k // per_group
        heads = tuple(i + group * r for i in _ranges(r, per_group, "query-head axis")[k % per_group])
        return heads, (group,)
    if cfg.variant == "mla":
        heads = _ranges(h, phi, "query-head axis")[k]
        return heads, [unit(-1, -1, heads)]
    if cfg.variant == "gla":  # tpsim.py:92-106: latent-group axis, then heads within a group
        g, r = cfg.g, h // cfg.g
        if phi <= g:
            us = [unit(j, -1, range(j * r, (j + 1) * r)) for j in _ranges(g, phi, "latent-group axis")[k]]
            return tuple(i for u in us for i in u[3]), us
        per_group = phi // g
        if phi % g != 0 or r % per_group != 0:
            raise OracleError(f"gla: cannot split {r} heads per group across {per_group} devices")
        group = k // per_group
        heads = tuple(i + group * r for i in _ranges(r, per_group, "query-head axis")[k % per_group])
        return heads, [unit(group, -1, heads)]
    if cfg.branches == 4:  # tpsim.py:108-116
        if phi <= 4:
            return all_heads, [unit(-1, b, all_heads) for b in _ranges(4, phi, "latent-block axis")[k]]
        block, half = k // 2, k % 2
        heads = _ranges(h, 2, "query-head axis")[half]
        return heads, [unit(-1, block, heads)]
    pairs = [(grp, b) for grp in range(2) for b in range(2)]  # mlra-2, tpsim.py:117-131
    half_heads = [tuple(range(grp * (h // 2), (grp + 1) * (h // 2))) for grp in range(2)]
    if phi == 1:
        return all_heads, [unit(grp, b, half_heads[grp]) for grp, b in pairs]
    if phi == 2:
        return half_heads[k], [unit(k, b, half_heads[k]) for b in range(2)]
    if phi == 4:
        grp, b = pairs[k]
        return half_heads[grp], [unit(grp, b, half_heads[grp])]
    grp, b = pairs[k // 2]
    heads = tuple(i + grp * (h // 2) for i in _ranges(h // 2, 2, "query-head axis")[k % 2])
    return heads, [unit(grp, b, heads)]


def sim_decode_attention(cfg: Cfg, w: dict, streams: dict, q_nope, q_rope, phi: int) -> tuple:
    """sim_decode's attention + reduction (attnkit/tpsim.py:253-286) over a complete cache.

    Returns (out, kind, per-device element reads). Devices read only the streams they own,
    and the reduction runs in device-id order (tpsim.py:275-276)."""
    contribs, reads = [], []
    for k in range(phi):
        heads, ulist = shard_units(cfg, phi, k)
        owned = {u[0]: streams[u[0]] for u in ulist}
        owned["rope"] = streams["rope"]
        cache = Cache(owned)
        contribs.extend(attend_latent(cfg, w, cache, q_nope, q_rope, ulist))
        reads.append(cache.reads)
    out, kind = reduce_contributions(cfg, contribs)
    return out, kind, reads


def per_device_load(cfg: Cfg, phi: int) -> Fraction:  # attnkit/costs.py:70-102 (served variants)
    if phi not in TP_DEGREES:
        raise OracleError(f"unsupported TP degree {phi}")
    if cfg.variant == "gqa":
        return Fraction(2 * cfg.g, min(phi, cfg.g))
    if cfg.variant == "mla":
        return Fraction(cfg.d_c + cfg.d_h_rope, cfg.d_h)
    if cfg.variant == "gla":
        return Fraction(cfg.d_c, min(phi, cfg.g) * cfg.d_h) + Fraction(cfg.d_h_rope, cfg.d_h)
    if cfg.variant == "mlra":
        return Fraction(cfg.d_c, min(phi, 4) * cfg.d_h) + Fraction(cfg.d_h_rope, cfg.d_h)
    raise OracleError(f"no loading rule for {cfg.variant}")


# ----------------------------------------------------------------------------- output side (8(f) row 2)
def sigmoid(x: np.ndarray) -> np.ndarray:  # attnkit/tensors.py:101-102
    return 1.0 / (1.0 + np.exp(-x))


def gated_output(hidden: np.ndarray, out_flat: np.ndarray, w_g: np.ndarray) -> np.ndarray:  # attnkit/zoo.py:125-127
    return out_flat * sigmoid(hidden @ w_g)


def attention_block_output(hidden: np.ndarray, out_flat: np.ndarray, w_o: np.ndarray, w_g=None) -> np.ndarray:
    """The attention half of attnkit/zoo.py:146-149 (block_forward): the gate is driven by the
    un-normalised block input, then hidden + gated @ w_o."""
    flat = gated_output(hidden, out_flat, w_g) if w_g is not None else out_flat
    return hidden + flat @ w_o


def tp_attention_block_output(hidden: np.ndarray, parts, w_o: np.ndarray, w_g, d_h: int) -> np.ndarray:
    """The same under tensor parallelism: parts = [(heads, out_r [n, len(heads)*d_h])] in device
    order (per-head contributions, summed like attnkit/decode.py:264-285); each device applies
    the gate and W_o to its columns and the [n, d] results are summed in device order."""
    acc = np.zeros((hidden.shape[0], w_o.shape[1]))
    for heads, out_r in parts:
        cols = np.concatenate([np.arange(i * d_h, (i + 1) * d_h) for i in heads])
        g = out_r * sigmoid(hidden @ w_g[:, cols]) if w_g is not None else out_r
        acc = acc + g @ w_o[cols]
    return hidden + acc


def max_rel_err(a: np.ndarray, b: np.ndarray) -> float:  # attnkit/selftest.py:101-103
    scale = max(float(np.max(np.abs(a))), 1e-30)
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float64 values to bfloat16 (round-to-nearest-even) and back to float64."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)
