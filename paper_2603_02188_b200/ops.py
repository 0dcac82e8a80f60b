"""Torch-facing wrappers over the C ABI: one function per kernel, stream-ordered on the
current torch CUDA stream, no host synchronisation.

Tensors are plain torch CUDA tensors (bf16 for cache / queries / weights, fp32 for
partials and outputs, int32 for page tables). Shapes follow include/mlra_b200.h.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .errors import ConfigError, ShapeMismatchError

LOG2E = 1.4426950408889634


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need(t: torch.Tensor, dtype, name: str, dim: int | None = None) -> None:
    if not t.is_cuda:
        raise ShapeMismatchError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ShapeMismatchError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ShapeMismatchError(f"{name} must be contiguous")
    if dim is not None and t.dim() != dim:
        raise ShapeMismatchError(f"{name} must be {dim}-D, got shape {tuple(t.shape)}")


def num_sms() -> int:
    return _lib.load().mlra_num_sms()


def default_splits(batch: int, max_seqlen: int, nb: int, sub: int, heads: int | None = None) -> int:
    """K2's split count: one wave of CTAs over the SMs (with ``heads``: counting K2's head groups)."""
    if heads is not None:
        return _lib.load().mlra_default_splits_heads(batch, max_seqlen, nb, sub, heads)
    return _lib.load().mlra_default_splits(batch, max_seqlen, nb, sub)


def cache_append(rows: torch.Tensor, block_table: torch.Tensor, positions: torch.Tensor, pool: torch.Tensor,
                 page_size: int, advance: bool = False) -> None:
    """K0: pool[page(pos), pos % page_size] = rows[s] for every sequence s; with ``advance``
    the kernel also bumps positions[s] (pass the sequence lengths: the reference append)."""
    _need(rows, torch.bfloat16, "rows", 2)
    _need(block_table, torch.int32, "block_table", 2)
    _need(positions, torch.int32, "positions", 1)
    _need(pool, torch.bfloat16, "pool", 2)
    B, W = rows.shape
    if pool.shape[1] != W:
        raise ShapeMismatchError(f"cache append: row width {W} != pool width {pool.shape[1]}")
    rc = _lib.load().mlra_cache_append(rows.data_ptr(), block_table.data_ptr(), positions.data_ptr(), B, W,
                                       page_size, block_table.shape[1], int(advance), pool.data_ptr(), _stream())
    _lib.check(rc, "mlra_cache_append")


def cache_append_latent(kv_raw: torch.Tensor, kr_raw: torch.Tensor, rope_pos: torch.Tensor | None,
                        slots: torch.Tensor | None,
                        block_table: torch.Tensor, pool: torch.Tensor, page_size: int, *, branches: int, block0: int,
                        nblocks: int, dlp: int, drp: int, alpha_kv: float, rope_base: float = 10000.0,
                        eps: float = 1e-6, norm_groups: int = 1, advance: bool = False,
                        chain: bool = False) -> None:
    """K0 fused: rmsnorm*alpha_kv of kv_raw [B, d_c] (owned blocks), rope of kr_raw [B, dr] at
    rope_pos (None: at the slot written), padded, appended as one bf16 pool row per sequence at
    slots[s] (then slots[s] += 1 with ``advance``). slots=None: the rows are one sequence's tokens
    0..B-1 (prefill), row s at slot s of block_table row 0. ``chain``: PDL launch that releases
    the next kernel at once -- only when that kernel waits for K0 before reading the pool."""
    _need(kv_raw, torch.float32, "kv_raw", 2)
    _need(kr_raw, torch.float32, "kr_raw", 2)
    if rope_pos is not None:
        _need(rope_pos, torch.int32, "rope_pos", 1)
    if slots is not None:
        _need(slots, torch.int32, "slots", 1)
    _need(block_table, torch.int32, "block_table", 2)
    _need(pool, torch.bfloat16, "pool", 2)
    B, d_c = kv_raw.shape
    dr = kr_raw.shape[1]
    if pool.shape[1] != nblocks * dlp + drp:
        raise ShapeMismatchError(f"cache_append_latent: pool width {pool.shape[1]} != {nblocks * dlp + drp}")
    rc = _lib.load().mlra_cache_append_latent(kv_raw.data_ptr(), kr_raw.data_ptr(),
                                              None if rope_pos is None else rope_pos.data_ptr(),
                                              None if slots is None else slots.data_ptr(), block_table.data_ptr(),
                                              B, d_c, branches, block0,
                                              nblocks, dlp, dr, drp, float(alpha_kv), float(rope_base), float(eps),
                                              page_size, block_table.shape[1], norm_groups,
                                              int(advance) | (2 if chain else 0),
                                              pool.data_ptr(), _stream())
    _lib.check(rc, "mlra_cache_append_latent")


def absorb_query(q_nope: torch.Tensor, q_rope: torch.Tensor, w_uk_packed: torch.Tensor, nb: int, dlat: int,
                 score_scale: float, out: tuple[torch.Tensor, torch.Tensor] | None = None):
    """K1: q_abs [B, NB, H, DLAT] and scaled q_rope [B, H, DR] (both bf16)."""
    _need(q_nope, torch.bfloat16, "q_nope", 3)
    _need(q_rope, torch.bfloat16, "q_rope", 3)
    _need(w_uk_packed, torch.bfloat16, "w_uk", 3)
    B, H, DH = q_nope.shape
    DR = q_rope.shape[2]
    if tuple(w_uk_packed.shape) != (H, DH, nb * dlat):
        raise ShapeMismatchError(f"w_uk packed shape {tuple(w_uk_packed.shape)} != {(H, DH, nb * dlat)}")
    if out is None:
        q_abs = torch.empty((B, nb, H, dlat), dtype=torch.bfloat16, device=q_nope.device)
        q_rs = torch.empty((B, H, DR), dtype=torch.bfloat16, device=q_nope.device)
    else:
        q_abs, q_rs = out
    rc = _lib.load().mlra_absorb_query(q_nope.data_ptr(), q_rope.data_ptr(), w_uk_packed.data_ptr(),
                                       q_abs.data_ptr(), q_rs.data_ptr(), B, H, DH, nb, dlat, DR,
                                       float(score_scale), _stream())
    _lib.check(rc, "mlra_absorb_query")
    return q_abs, q_rs


def decode_partials(q_abs: torch.Tensor, q_rope: torch.Tensor, pool: torch.Tensor, block_table: torch.Tensor,
                    seqlens: torch.Tensor, page_size: int, nb: int, sub: int, dls: int, nsplit: int,
                    out: tuple[torch.Tensor, torch.Tensor] | None = None):
    """K2: split-KV partials (o_part [B, nsplit, NB, H, DLAT], lse_part [B, nsplit, NB, H])."""
    _need(q_abs, torch.bfloat16, "q_abs", 4)
    _need(q_rope, torch.bfloat16, "q_rope", 3)
    _need(pool, torch.bfloat16, "pool", 2)
    _need(block_table, torch.int32, "block_table", 2)
    _need(seqlens, torch.int32, "seqlens", 1)
    B, NB, H, DLAT = q_abs.shape
    DR = q_rope.shape[2]
    if NB != nb or DLAT != sub * dls:
        raise ShapeMismatchError(f"q_abs shape {tuple(q_abs.shape)} inconsistent with nb={nb} sub={sub} dls={dls}")
    W = nb * DLAT + DR
    if pool.shape[1] != W or pool.shape[0] % page_size:
        raise ShapeMismatchError(f"pool shape {tuple(pool.shape)} inconsistent with row width {W}/page {page_size}")
    if out is None:
        o_part = torch.empty((B, nsplit, NB, H, DLAT), dtype=torch.float32, device=q_abs.device)
        lse_part = torch.empty((B, nsplit, NB, H), dtype=torch.float32, device=q_abs.device)
    else:
        o_part, lse_part = out
    rc = _lib.load().mlra_decode_partials(q_abs.data_ptr(), q_rope.data_ptr(), pool.data_ptr(),
                                          block_table.data_ptr(), seqlens.data_ptr(), o_part.data_ptr(),
                                          lse_part.data_ptr(), B, H, NB, sub, dls, DR, page_size,
                                          block_table.shape[1], pool.shape[0] // page_size, nsplit, _stream())
    _lib.check(rc, "mlra_decode_partials")
    return o_part, lse_part


_STATUS: dict = {}


def status_word(device) -> torch.Tensor:
    """Per-device int32 numeric status word for the stand-alone K3 calls (``combine``)."""
    key = str(torch.device(device))
    if key not in _STATUS:
        _STATUS[key] = torch.zeros(1, dtype=torch.int32, device=device)
    return _STATUS[key]


def check_status(status: torch.Tensor, what: str = "decode") -> None:
    """Synchronise the current stream, read and reset a status word; NumericError if the merge
    flagged a NaN logit or a row with no finite logit (attnkit/tensors.py:74-78)."""
    rc = _lib.load().mlra_check_status(status.data_ptr(), 1, _stream())
    _lib.check(rc, what)


def combine(o_part: torch.Tensor, lse_part: torch.Tensor, w_uv_packed: torch.Tensor | None, alpha: float,
            out: torch.Tensor | None = None, per_branch: bool = False, scratch: torch.Tensor | None = None,
            status: torch.Tensor | None = None):
    """K3: merge splits; with w_uv_packed [H, NB*DLAT, DH] also up-project (summing branches,
    or per branch when ``per_branch``). Numeric flags go to ``status`` (default: the device's
    status word, see ``check_status``)."""
    _need(o_part, torch.float32, "o_part", 5)
    _need(lse_part, torch.float32, "lse_part", 4)
    B, nsplit, NB, H, DLAT = o_part.shape
    mode = 0
    if w_uv_packed is not None:
        _need(w_uv_packed, torch.bfloat16, "w_uv", 3)
        DH = w_uv_packed.shape[2]
        if tuple(w_uv_packed.shape[:2]) != (H, NB * DLAT):
            raise ShapeMismatchError(f"w_uv packed shape {tuple(w_uv_packed.shape)} != {(H, NB * DLAT, DH)}")
        mode = 2 if per_branch else 1
        shape = (B, NB, H, DH) if per_branch else (B, H, DH)
        if scratch is None:
            scratch = torch.empty((B, H, NB * DLAT), dtype=torch.float32, device=o_part.device)
    else:
        DH = DLAT
        shape = (B, NB, H, DLAT)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=o_part.device)
    rc = _lib.load().mlra_combine(o_part.data_ptr(), lse_part.data_ptr(),
                                  w_uv_packed.data_ptr() if mode else None, out.data_ptr(),
                                  scratch.data_ptr() if mode else None, B, H, NB, DLAT, DH, nsplit, float(alpha),
                                  mode, (status if status is not None else status_word(o_part.device)).data_ptr(),
                                  _stream())
    _lib.check(rc, "mlra_combine")
    return out


class DecodeWorkspace:
    """Device scratch for one fused decode step (sized by mlra_workspace_bytes)."""

    def __init__(self, batch: int, heads: int, nb: int, dlat: int, dr: int, nsplit: int, device):
        nbytes = _lib.load().mlra_workspace_bytes(batch, heads, nb, dlat, dr, nsplit)
        self.key = (batch, heads, nb, dlat, dr, nsplit)
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)  # counters and status start at 0
        self.status = self.buf[:4].view(torch.int32)  # numeric status word (include/mlra_b200.h)


def decode_step(q_nope, q_rope, w_uk_packed, w_uv_packed, pool, block_table, seqlens, page_size: int, nb: int,
                sub: int, dls: int, nsplit: int, score_scale: float, alpha: float, workspace: DecodeWorkspace,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """K1 + K2 + K3 through the single C-ABI entry point mlra_decode_step. ``w_uk_packed=None``:
    q_nope is the pre-absorbed, pre-scaled q~ [B, NB, H, DLAT] (K-1 with the pre-multiplied
    weight) and q_rope is pre-scaled; the step is K2 + K3."""
    if w_uk_packed is None:
        B, _, H, _ = q_nope.shape
        DH = w_uv_packed.shape[2]
    else:
        B, H, DH = q_nope.shape
    DR = q_rope.shape[2]
    dlat = sub * dls
    if workspace.key != (B, H, nb, dlat, DR, nsplit):
        raise ConfigError(f"workspace sized for {workspace.key}, call needs {(B, H, nb, dlat, DR, nsplit)}")
    if out is None:
        out = torch.empty((B, H, DH), dtype=torch.float32, device=q_nope.device)
    rc = _lib.load().mlra_decode_step(q_nope.data_ptr(), q_rope.data_ptr(),
                                      None if w_uk_packed is None else w_uk_packed.data_ptr(),
                                      w_uv_packed.data_ptr(), pool.data_ptr(), block_table.data_ptr(),
                                      seqlens.data_ptr(), out.data_ptr(), workspace.buf.data_ptr(), B, H, DH, nb,
                                      sub, dls, DR, page_size, block_table.shape[1], pool.shape[0] // page_size,
                                      nsplit, float(score_scale), float(alpha), _stream())
    _lib.check(rc, "mlra_decode_step")
    return out


def decode_step_ragged(q_nope, q_rope, w_uk_packed, w_uv_packed, pool, block_table, seqlens, page_size: int, nb: int,
                       sub: int, dls: int, nsplit_max: int, score_scale: float, alpha: float,
                       workspace: DecodeWorkspace, out: torch.Tensor | None = None) -> torch.Tensor:
    """decode_step for ragged batches (mlra_decode_step_ragged): the device-side plan balances the
    sequences' token tiles over one wave of K2 CTAs (up to nsplit_max splits per sequence)."""
    if w_uk_packed is None:
        B, _, H, _ = q_nope.shape
        DH = w_uv_packed.shape[2]
    else:
        B, H, DH = q_nope.shape
    DR = q_rope.shape[2]
    dlat = sub * dls
    if workspace.key != (B, H, nb, dlat, DR, nsplit_max):
        raise ConfigError(f"workspace sized for {workspace.key}, call needs {(B, H, nb, dlat, DR, nsplit_max)}")
    if out is None:
        out = torch.empty((B, H, DH), dtype=torch.float32, device=q_nope.device)
    rc = _lib.load().mlra_decode_step_ragged(q_nope.data_ptr(), q_rope.data_ptr(),
                                             None if w_uk_packed is None else w_uk_packed.data_ptr(),
                                             w_uv_packed.data_ptr(), pool.data_ptr(), block_table.data_ptr(),
                                             seqlens.data_ptr(), out.data_ptr(), workspace.buf.data_ptr(), B, H, DH,
                                             nb, sub, dls, DR, page_size, block_table.shape[1],
                                             pool.shape[0] // page_size, nsplit_max, float(score_scale),
                                             float(alpha), _stream())
    _lib.check(rc, "mlra_decode_step_ragged")
    return out


def decode_step_tp(q_nope, q_rope, w_uk_packed, w_uv_packed, pool, block_table, seqlens, page_size: int, nb: int,
                   sub: int, dls: int, nsplit: int, score_scale: float, alpha: float, workspace: DecodeWorkspace,
                   rank: int, world: int, comm_ptrs, out: torch.Tensor | None = None,
                   comm_n: int | None = None) -> torch.Tensor:
    """decode_step with the sum over the TP ranks fused into K3 (mlra_decode_step_tp): every rank
    gets the device-order sum of all ranks' outputs. comm_ptrs: the ranks' allreduce regions
    (collective.PeerAllReduce(group, B*H*DH).ptrs)."""
    B, H, DH = q_nope.shape
    DR = q_rope.shape[2]
    dlat = sub * dls
    if workspace.key != (B, H, nb, dlat, DR, nsplit):
        raise ConfigError(f"workspace sized for {workspace.key}, call needs {(B, H, nb, dlat, DR, nsplit)}")
    if world > 1 and comm_n is not None and comm_n != B * H * DH:
        # the fused epilogue derives the receive stride, flag array and epoch counter of the
        # regions from B*H*DH: a region sized for another n would be read and written off-layout
        raise ConfigError(f"peer regions sized for {comm_n} values, the step reduces {B * H * DH}")
    if out is None:
        out = torch.empty((B, H, DH), dtype=torch.float32, device=q_nope.device)
    elif out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != (B, H, DH):
        raise ShapeMismatchError(f"out must be a contiguous float32 [{B}, {H}, {DH}] tensor")
    rc = _lib.load().mlra_decode_step_tp(q_nope.data_ptr(), q_rope.data_ptr(), w_uk_packed.data_ptr(),
                                         w_uv_packed.data_ptr(), pool.data_ptr(), block_table.data_ptr(),
                                         seqlens.data_ptr(), out.data_ptr(), workspace.buf.data_ptr(), B, H, DH, nb,
                                         sub, dls, DR, page_size, block_table.shape[1], pool.shape[0] // page_size,
                                         nsplit, float(score_scale), float(alpha), rank, world,
                                         _ptr_array(comm_ptrs) if world > 1 else None, _stream())
    _lib.check(rc, "mlra_decode_step_tp")
    return out


# ----------------------------------------------------------------------------- GQA variant
def gqa_default_splits(batch: int, kv_heads: int, max_seqlen: int) -> int:
    return _lib.load().mlra_gqa_default_splits(batch, kv_heads, max_seqlen)


def gqa_decode_partials(q: torch.Tensor, pool: torch.Tensor, block_table: torch.Tensor, seqlens: torch.Tensor,
                        page_size: int, nsplit: int, score_scale: float, out=None):
    """K2 (GQA): q [B, G, R, DH] bf16 (post-RoPE, unscaled, DH in {64, 128}) over a pool of rows
    [K_0..K_{G-1} | V_0..V_{G-1}] -> o_part [B, nsplit, G, R, DH], lse_part [B, nsplit, G, R]."""
    _need(q, torch.bfloat16, "q", 4)
    _need(pool, torch.bfloat16, "pool", 2)
    _need(block_table, torch.int32, "block_table", 2)
    _need(seqlens, torch.int32, "seqlens", 1)
    B, G, R, DH = q.shape
    if pool.shape[1] != 2 * G * DH:
        raise ShapeMismatchError(f"gqa pool width {pool.shape[1]} != 2*G*DH = {2 * G * DH}")
    if out is None:
        o_part = torch.empty((B, nsplit, G, R, DH), dtype=torch.float32, device=q.device)
        lse_part = torch.empty((B, nsplit, G, R), dtype=torch.float32, device=q.device)
    else:
        o_part, lse_part = out
    rc = _lib.load().mlra_gqa_decode_partials(q.data_ptr(), pool.data_ptr(), block_table.data_ptr(),
                                              seqlens.data_ptr(), o_part.data_ptr(), lse_part.data_ptr(), B, G, R,
                                              DH, page_size, block_table.shape[1], pool.shape[0] // page_size, nsplit,
                                              float(score_scale), _stream())
    _lib.check(rc, "mlra_gqa_decode_partials")
    return o_part, lse_part


class GqaWorkspace:
    """Device scratch (split partials) of one GQA decode step."""

    def __init__(self, batch: int, kv_heads: int, reps: int, dh: int, nsplit: int, device):
        nbytes = _lib.load().mlra_gqa_workspace_bytes(batch, kv_heads, reps, dh, nsplit)
        self.key = (batch, kv_heads, reps, dh, nsplit)
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.status = self.buf[:4].view(torch.int32)  # numeric status word


def gqa_decode_step(q: torch.Tensor, pool: torch.Tensor, block_table: torch.Tensor, seqlens: torch.Tensor,
                    page_size: int, nsplit: int, score_scale: float, workspace: GqaWorkspace,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """K2 (GQA) + split merge: q [B, G, R, DH] -> out [B, G*R, DH] fp32 (head b*R + j)."""
    _need(q, torch.bfloat16, "q", 4)
    B, G, R, DH = q.shape
    if workspace.key != (B, G, R, DH, nsplit):
        raise ConfigError(f"gqa workspace sized for {workspace.key}, call needs {(B, G, R, DH, nsplit)}")
    if out is None:
        out = torch.empty((B, G * R, DH), dtype=torch.float32, device=q.device)
    rc = _lib.load().mlra_gqa_decode_step(q.data_ptr(), pool.data_ptr(), block_table.data_ptr(), seqlens.data_ptr(),
                                          out.data_ptr(), workspace.buf.data_ptr(), B, G, R, DH, page_size,
                                          block_table.shape[1], pool.shape[0] // page_size, nsplit, float(score_scale),
                                          _stream())
    _lib.check(rc, "mlra_gqa_decode_step")
    return out


def score_scale(tau: float) -> float:
    """Scale folded into the queries: scores are evaluated in the log2 domain."""
    return float(tau) * LOG2E


def latent_geometry(dlat: int) -> tuple[int, int]:
    """(SUB, DLS): split a branch latent of width dlat into sub-blocks of 128 (or 64)."""
    if dlat % 128 == 0:
        return dlat // 128, 128
    if dlat == 64:
        return 1, 64
    raise ConfigError(f"latent width {dlat} per branch must be 64 or a multiple of 128")


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("math", "torch")]


# ----------------------------------------------------------------------------- K4: output side
def outproj_comm_bytes(batch: int, d: int, world: int) -> int:
    return int(_lib.load().mlra_outproj_comm_bytes(batch, d, world))


def _ptr_array(ptrs):
    import ctypes

    arr = (ctypes.c_void_p * len(ptrs))(*[int(p) if p is not None else None for p in ptrs])
    return arr


def _outproj_shapes(attn, gate_pre, w_o, resid, y):
    _need(attn, torch.float32, "attn", 2)
    _need(w_o, torch.bfloat16, "w_o", 2)
    _need(y, torch.float32, "y", 2)
    B, K = attn.shape
    D = w_o.shape[1]
    if w_o.shape[0] != K:
        raise ShapeMismatchError(f"outproj: w_o rows {w_o.shape[0]} != attention width {K}")
    if tuple(y.shape) != (B, D):
        raise ShapeMismatchError(f"outproj: y {tuple(y.shape)} != {(B, D)}")
    if gate_pre is not None:
        _need(gate_pre, torch.float32, "gate_pre", 2)
        if gate_pre.shape != attn.shape:
            raise ShapeMismatchError(f"outproj: gate_pre {tuple(gate_pre.shape)} != attn {tuple(attn.shape)}")
    if resid is not None:
        _need(resid, torch.float32, "resid", 2)
        if tuple(resid.shape) != (B, D):
            raise ShapeMismatchError(f"outproj: resid {tuple(resid.shape)} != {(B, D)}")
    return B, K, D


def outproj_workspace(batch: int, k: int, device) -> torch.Tensor:
    return torch.empty(int(_lib.load().mlra_outproj_workspace_bytes(batch, k)), dtype=torch.uint8, device=device)


def outproj(attn: torch.Tensor, gate_pre: torch.Tensor | None, w_o: torch.Tensor, resid: torch.Tensor | None,
            y: torch.Tensor, rank: int = 0, world: int = 1, comm_ptrs=None,
            workspace: torch.Tensor | None = None) -> torch.Tensor:
    """K4a + K4: y = resid + sum over ranks of (attn * sigmoid(gate_pre)) @ w_o (zoo.py:125-149).
    world > 1: comm_ptrs = every rank's communication region as mapped here."""
    B, K, D = _outproj_shapes(attn, gate_pre, w_o, resid, y)
    ws = workspace if workspace is not None else outproj_workspace(B, K, attn.device)
    if ws.numel() < _lib.load().mlra_outproj_workspace_bytes(B, K):
        raise ShapeMismatchError("outproj: workspace too small")
    comm = _ptr_array(comm_ptrs) if comm_ptrs is not None else None
    rc = _lib.load().mlra_outproj(attn.data_ptr(), _lib.ptr(gate_pre), w_o.data_ptr(), _lib.ptr(resid), y.data_ptr(),
                                  B, K, D, rank, world, comm, ws.data_ptr(), _stream())
    _lib.check(rc, "mlra_outproj")
    return y


def outproj_sim(attns, gates, w_os, resid, ys, comms) -> None:
    """K4 with len(attns) ranks simulated on one device (tests): per-rank lists of tensors,
    comms = per-rank communication regions (uint8 CUDA tensors of outproj_comm_bytes)."""
    world = len(attns)
    B, K, D = _outproj_shapes(attns[0], None if gates is None else gates[0], w_os[0], resid, ys[0])
    for r in range(world):
        _outproj_shapes(attns[r], None if gates is None else gates[r], w_os[r], resid, ys[r])
        if comms[r].numel() < outproj_comm_bytes(B, D, world):
            raise ShapeMismatchError("outproj_sim: communication region too small")
    wss = [outproj_workspace(B, K, attns[0].device) for _ in range(world)]
    rc = _lib.load().mlra_outproj_sim(_ptr_array([a.data_ptr() for a in attns]),
                                      None if gates is None else _ptr_array([g.data_ptr() for g in gates]),
                                      _ptr_array([w.data_ptr() for w in w_os]), _lib.ptr(resid),
                                      _ptr_array([y.data_ptr() for y in ys]), B, K, D, world,
                                      _ptr_array([c.data_ptr() for c in comms]),
                                      _ptr_array([w.data_ptr() for w in wss]), _stream())
    _lib.check(rc, "mlra_outproj_sim")


def comm_alloc(nbytes: int) -> int:
    """Zero-filled device allocation of its own (exact IPC mapping); returns the pointer."""
    import ctypes

    out = ctypes.c_void_p()
    _lib.check(_lib.load().mlra_comm_alloc(nbytes, ctypes.byref(out)), "mlra_comm_alloc")
    return int(out.value)


def comm_free(ptr: int) -> None:
    _lib.check(_lib.load().mlra_comm_free(ptr), "mlra_comm_free")


def ipc_handle(ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a comm_alloc allocation."""
    import ctypes

    buf = ctypes.create_string_buffer(64)
    _lib.check(_lib.load().mlra_ipc_handle(ptr, buf), "mlra_ipc_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    import ctypes

    if len(handle) != 64:
        raise ConfigError(f"ipc_open: handle of {len(handle)} bytes, expected 64")
    out = ctypes.c_void_p()
    _lib.check(_lib.load().mlra_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(out)), "mlra_ipc_open")
    return int(out.value)


def ipc_close(ptr: int) -> None:
    _lib.check(_lib.load().mlra_ipc_close(ptr), "mlra_ipc_close")


# ----------------------------------------------------------------------------- K5: peer all-reduce
def allreduce_comm_bytes(n: int, world: int) -> int:
    return int(_lib.load().mlra_allreduce_comm_bytes(n, world))


def allreduce(x: torch.Tensor, y: torch.Tensor, rank: int, world: int, comm_ptrs) -> torch.Tensor:
    """K5: y = sum over ranks of x (ascending rank order) through the peer regions comm_ptrs."""
    _need(x, torch.float32, "x")
    _need(y, torch.float32, "y")
    if x.numel() != y.numel():
        raise ShapeMismatchError(f"allreduce: x has {x.numel()} values, y {y.numel()}")
    rc = _lib.load().mlra_allreduce(x.data_ptr(), y.data_ptr(), x.numel(), rank, world, _ptr_array(comm_ptrs),
                                    _stream())
    _lib.check(rc, "mlra_allreduce")
    return y


def allreduce_sim(xs, ys, comms) -> None:
    """K5 with len(xs) ranks simulated on one device (tests); comms: uint8 CUDA tensors."""
    world = len(xs)
    n = xs[0].numel()
    for x, y, c in zip(xs, ys, comms):
        _need(x, torch.float32, "x")
        _need(y, torch.float32, "y")
        if x.numel() != n or y.numel() != n or c.numel() < allreduce_comm_bytes(n, world):
            raise ShapeMismatchError("allreduce_sim: inconsistent sizes")
    rc = _lib.load().mlra_allreduce_sim(_ptr_array([x.data_ptr() for x in xs]), _ptr_array([y.data_ptr() for y in ys]),
                                        n, world, _ptr_array([c.data_ptr() for c in comms]), _stream())
    _lib.check(rc, "mlra_allreduce_sim")



# ----------------------------------------------------------------------------- K-1 projections
def slab_shape(K: int, N: int) -> tuple[int, int, int]:
    return (-(-N // 64), -(-K // 64) * 64, 64)


def slab_pack(w: torch.Tensor) -> torch.Tensor:
    """[K, N] weight -> the K-1 kernels' slab-packed bf16 [ceil(N/64)][round_up(K, 64)][64]:
    element [s][k][c] = w[k][64 s + c] (zero outside w; include/mlra_b200.h)."""
    K, N = w.shape
    ns, kp, _ = slab_shape(K, N)
    full = torch.zeros((kp, ns * 64), dtype=torch.bfloat16, device=w.device)
    full[:K, :N] = w.to(torch.bfloat16)
    return full.reshape(kp, ns, 64).permute(1, 0, 2).contiguous()


def proj_down(x: torch.Tensor, w: torch.Tensor, n_q: int, n_kv: int, n_kr: int, c_q_raw: torch.Tensor | None,
              kv_raw: torch.Tensor | None, kr_raw: torch.Tensor | None, ssq: torch.Tensor | None) -> None:
    """K-1 down: [c_q_raw | kv_raw | kr_raw] = x . W  (x [M, K] fp32, w = ``slab_pack(W)`` of the
    bf16 [K, n_q+n_kv+n_kr] weight), plus the per-64-column sums of squares of c_q_raw into ssq
    [ceil(n_q/64), M]."""
    _need(x, torch.float32, "x", 2)
    _need(w, torch.bfloat16, "w", 3)
    M, K = x.shape
    if tuple(w.shape) != slab_shape(K, n_q + n_kv + n_kr):
        raise ShapeMismatchError(f"proj_down: w {tuple(w.shape)} is not the slab pack of [{K}, {n_q}+{n_kv}+{n_kr}]")
    outs = []
    for t, width, name in ((c_q_raw, n_q, "c_q_raw"), (kv_raw, n_kv, "kv_raw"), (kr_raw, n_kr, "kr_raw")):
        if t is not None:
            _need(t, torch.float32, name, 2)
            if tuple(t.shape) != (M, width):
                raise ShapeMismatchError(f"proj_down: {name} {tuple(t.shape)} != {(M, width)}")
        outs.append(0 if t is None else t.data_ptr())
    if ssq is not None:
        _need(ssq, torch.float32, "ssq", 2)
        if tuple(ssq.shape) != (-(-n_q // 64), M):
            raise ShapeMismatchError(f"proj_down: ssq {tuple(ssq.shape)} != {(-(-n_q // 64), M)}")
    rc = _lib.load().mlra_proj_down(x.data_ptr(), w.data_ptr(), M, K, n_q, n_kv, n_kr, *outs,
                                    0 if ssq is None else ssq.data_ptr(), _stream())
    _lib.check(rc, "mlra_proj_down")


def proj_query(c_q_raw: torch.Tensor, ssq: torch.Tensor | None, alpha_q: float, w: torch.Tensor, nq: int, heads: int,
               dr: int, pos: torch.Tensor, q_out: torch.Tensor, r_out: torch.Tensor, *, q_scale: float = 1.0,
               r_scale: float = 1.0, eps: float = 1e-6, rope_base: float = 10000.0, pos_delta: int = 0) -> None:
    """K-1 query: c_q = alpha_q * rmsnorm(c_q_raw) (statistics from ssq), [q_x | q_r] = c_q . w;
    q_out [M, nq] bf16 = q_scale * q_x, r_out [M, heads, drp] bf16 = r_scale * rope(q_r, pos + pos_delta)."""
    _need(c_q_raw, torch.float32, "c_q_raw", 2)
    _need(w, torch.bfloat16, "w", 3)
    _need(pos, torch.int32, "pos", 1)
    _need(q_out, torch.bfloat16, "q_out")
    _need(r_out, torch.bfloat16, "r_out", 3)
    M, K = c_q_raw.shape
    if tuple(w.shape) != slab_shape(K, nq + heads * dr):
        raise ShapeMismatchError(f"proj_query: w {tuple(w.shape)} is not the slab pack of [{K}, {nq}+{heads}*{dr}]")
    if q_out.numel() != M * nq or r_out.shape[0] != M or r_out.shape[1] != heads or r_out.shape[2] < dr:
        raise ShapeMismatchError("proj_query: output shapes do not match")
    if pos.shape[0] < M:
        raise ShapeMismatchError(f"proj_query: {pos.shape[0]} positions for {M} rows")
    if ssq is not None:
        _need(ssq, torch.float32, "ssq", 2)
    rc = _lib.load().mlra_proj_query(c_q_raw.data_ptr(), 0 if ssq is None else ssq.data_ptr(), float(alpha_q),
                                     float(eps), w.data_ptr(), M, K, nq, heads, dr, r_out.shape[2], pos.data_ptr(),
                                     int(pos_delta), float(rope_base), float(q_scale), float(r_scale), q_out.data_ptr(),
                                     r_out.data_ptr(), _stream())
    _lib.check(rc, "mlra_proj_query")


def prefill_attention(q_abs: torch.Tensor, q_rope: torch.Tensor, w_uv_packed: torch.Tensor, pool: torch.Tensor,
                      block_table: torch.Tensor, page_size: int, nb: int, dlat: int, dr: int, alpha: float,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """K6: causal prefill attention of one sequence of n tokens already in the paged cache
    (block_table row 0): q_abs head-major [H, n, NB, DLAT] / q_rope [n, H, DRq] (pre-scaled by
    tau*log2e), w_uv [H, NB*DLAT, DH] -> out [n, H, DH] fp32 (alpha-scaled, branch-summed)."""
    _need(q_abs, torch.bfloat16, "q_abs", 4)
    _need(q_rope, torch.bfloat16, "q_rope", 3)
    _need(w_uv_packed, torch.bfloat16, "w_uv", 3)
    _need(pool, torch.bfloat16, "pool", 2)
    _need(block_table, torch.int32, "block_table", 2)
    H, n, NB, DLAT = q_abs.shape
    DH = w_uv_packed.shape[2]
    if NB != nb or DLAT != dlat or q_rope.shape[:2] != (n, H):
        raise ShapeMismatchError("prefill_attention: query shapes do not match")
    if out is None:
        out = torch.empty((n, H, DH), dtype=torch.float32, device=q_abs.device)
    rc = _lib.load().mlra_prefill_attention(q_abs.data_ptr(), q_rope.data_ptr(), w_uv_packed.data_ptr(),
                                            pool.data_ptr(), block_table.data_ptr(), out.data_ptr(), n, H, NB, DLAT,
                                            DH, dr, pool.shape[1] - NB * DLAT, q_rope.shape[2], page_size,
                                            block_table.shape[1],
                                            pool.shape[0] // page_size, float(alpha), _stream())
    _lib.check(rc, "mlra_prefill_attention")
    return out


def rows_split(x: torch.Tensor, K: int, norm: bool = False, alpha: float = 1.0, eps: float = 1e-6,
               stacked: bool = False):
    """x [n, >= K] fp32 (first K columns) -> (hi, lo) bf16 [n, K]: x or alpha * rmsnorm(x);
    ``stacked``: one [n, 2K] tensor [hi | lo] (the operand of a single GEMM against [W; W])."""
    _need(x, torch.float32, "x", 2)
    n = x.shape[0]
    if stacked:
        both = torch.empty((n, 2 * K), dtype=torch.bfloat16, device=x.device)
        hi_p, lo_p, ld = both.data_ptr(), both.data_ptr() + K * 2, 2 * K
    else:
        hi = torch.empty((n, K), dtype=torch.bfloat16, device=x.device)
        lo = torch.empty_like(hi)
        hi_p, lo_p, ld = hi.data_ptr(), lo.data_ptr(), K
    rc = _lib.load().mlra_rows_split(x.data_ptr(), n, K, x.shape[1], int(norm), float(alpha), float(eps), hi_p, lo_p,
                                     ld, _stream())
    _lib.check(rc, "mlra_rows_split")
    return both if stacked else (hi, lo)


def query_epilogue(y: torch.Tensor, nq: int, heads: int, dr: int, drq: int, pos0: int, q_scale: float = 1.0,
                   r_scale: float = 1.0, rope_base: float = 10000.0):
    """y [n, >= nq + heads*dr] fp32 -> (q bf16 [n, nq] * q_scale, rope(q_r) * r_scale bf16 [n, heads, drq])."""
    _need(y, torch.float32, "y", 2)
    n = y.shape[0]
    q = torch.empty((n, nq), dtype=torch.bfloat16, device=y.device)
    r = torch.empty((n, heads, drq), dtype=torch.bfloat16, device=y.device)
    rc = _lib.load().mlra_query_epilogue(y.data_ptr(), n, y.shape[1], nq, heads, dr, drq, int(pos0),
                                         float(rope_base), float(q_scale), float(r_scale), q.data_ptr(),
                                         r.data_ptr(), _stream())
    _lib.check(rc, "mlra_query_epilogue")
    return q, r
