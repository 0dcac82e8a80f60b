"""Pre-attention projections on the GPU: the rows a decode step appends and the queries it
attends with (attnkit/latent.py:129-159 latent_projections, attnkit/zoo.py:53-58 for gqa).

``KernelProjector`` is the decode path: the hand-written K-1 kernels
(csrc/proj_kernel.cuh) stream the bf16 weights once per step for a batch of <= 16 rows per
launch. ``LatentProjector`` / ``GqaProjector`` (torch, fp32 GEMMs) serve the many-row prefill
(real GEMMs: cuBLAS) and the gqa comparison variant.
"""

from __future__ import annotations

import torch

from . import ops
from .config import AttnConfig
from .errors import ShapeMismatchError
from .costs import calib_factors


def rmsnorm(x: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + eps)


def rope_rotate(x: torch.Tensor, positions: torch.Tensor, base: float = 10000.0) -> torch.Tensor:
    """Interleaved-pair RoPE (2l, 2l+1), theta_l = base^(-2l/dim) (attnkit/rope.py:36-66).
    x: [n, ..., dim]; positions: [n]."""
    dim = x.shape[-1]
    ell = torch.arange(dim // 2, dtype=torch.float64, device=x.device)
    freqs = float(base) ** (-2.0 * ell / dim)
    ang = positions.to(torch.float64)[:, None] * freqs[None, :]
    ang = ang.reshape((x.shape[0],) + (1,) * (x.ndim - 2) + (dim // 2,))
    cos, sin = torch.cos(ang).to(x.dtype), torch.sin(ang).to(x.dtype)
    even, odd = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = even * cos - odd * sin
    out[..., 1::2] = even * sin + odd * cos
    return out


class LatentProjector:
    """Device copies (fp32) of the projection weights of one WeightSet."""

    def __init__(self, cfg: AttnConfig, w, device):
        self.cfg = cfg
        f = lambda name: torch.as_tensor(w[name], dtype=torch.float32, device=device)  # noqa: E731
        self.w_dq, self.w_uq, self.w_qr, self.w_kr = f("w_dq"), f("w_uq"), f("w_qr"), f("w_kr")
        # every raw down-projection by name (w_dkv, or w_dkv_<j> per latent group)
        names = list(w.tensors) if hasattr(w, "tensors") else list(w.keys())  # WeightSet or plain dict
        self.w = {n: f(n) for n in names if str(n).startswith("w_dkv")}
        self.w_dkv = self.w.get("w_dkv")
        sf = calib_factors(cfg)
        self.alpha_q, self.alpha_kv = sf.alpha_q, sf.alpha_kv

    def queries(self, hidden: torch.Tensor, positions: torch.Tensor):
        """hidden [n, d] fp32 -> q_nope [n,h,d_h], q_rope [n,h,dr] (latent.py:134-139)."""
        cfg = self.cfg
        n = hidden.shape[0]
        c_q = self.alpha_q * rmsnorm(hidden @ self.w_dq)
        q_nope = (c_q @ self.w_uq).reshape(n, cfg.h, cfg.d_h)
        q_rope = rope_rotate((c_q @ self.w_qr).reshape(n, cfg.h, cfg.d_h_rope), positions)
        return q_nope, q_rope

    def __call__(self, hidden: torch.Tensor, positions: torch.Tensor):
        """hidden [n, d] fp32 -> q_nope [n,h,d_h], q_rope [n,h,dr], k_rope [n,dr], c_kv [n,d_c]."""
        cfg = self.cfg
        n = hidden.shape[0]
        c_q = self.alpha_q * rmsnorm(hidden @ self.w_dq)
        q_nope = (c_q @ self.w_uq).reshape(n, cfg.h, cfg.d_h)
        q_rope = rope_rotate((c_q @ self.w_qr).reshape(n, cfg.h, cfg.d_h_rope), positions)
        k_rope = rope_rotate(hidden @ self.w_kr, positions)
        c_kv = self.alpha_kv * rmsnorm(hidden @ self.w_dkv) if self.w_dkv is not None else None
        return q_nope, q_rope, k_rope, c_kv


class GqaProjector:
    def __init__(self, cfg: AttnConfig, w, device):
        self.cfg = cfg
        f = lambda name: torch.as_tensor(w[name], dtype=torch.float32, device=device)  # noqa: E731
        self.w_q, self.w_k, self.w_v = f("w_q"), f("w_k"), f("w_v")

    def __call__(self, hidden: torch.Tensor, positions: torch.Tensor):
        cfg = self.cfg
        n = hidden.shape[0]
        q = rope_rotate((hidden @ self.w_q).reshape(n, cfg.h, cfg.d_h), positions)
        k = rope_rotate((hidden @ self.w_k).reshape(n, cfg.g, cfg.d_h), positions)
        v = (hidden @ self.w_v).reshape(n, cfg.g, cfg.d_h)
        return q, k, v


def _gemm2(hilo: torch.Tensor, w2: torch.Tensor) -> torch.Tensor:
    """[hi | lo] [M, 2K] (bf16 planes of fp32 activations) times [W; W] [2K, N] bf16: ONE cuBLAS
    bf16 GEMM with fp32 accumulation and output (= (hi + lo) . W)."""
    return torch.mm(hilo, w2, out_dtype=torch.float32)


class KernelProjector:
    """K-1 on the GPU: the pre-attention projections of latent.py:129-159 as the hand-written
    weight-streaming GEMMs of csrc/proj_kernel.cuh (``ops.proj_down`` / ``ops.proj_query``).

    Packs once per (config, weights, owner), bf16, row-major (in, out), plus the slab packs
    (``ops.slab_pack``) the kernels stream:
      w_down  = [W^DQ | W^DKV_* (kv_names, concatenated) | W^KR]            (d, n_q + n_kv + n_kr)
      w_query = [W^Q | W^QR over the owner's heads]                          (d_cq, nq + H*dr)
    with W^Q = W^UQ (q_nope for K1: ``absorbed=False``) or, when ``absorbed``, the
    pre-multiplied W^UQ_(h) . W^UK_(b),(h)^T columns in (branch, head, latent) order, so the
    query kernel writes K2's absorbed query q~ directly (PAPER.md:84-94 Step 1 folded into the
    projection; tau*log2e applied in its epilogue) and K1 is skipped. ``absorbed=None`` picks
    it when the pre-multiplied weight is no larger than W^UQ (one latent block per device: an
    MLRA-4 / MLRA-2 TP4 rank).
    """

    def __init__(self, cfg: AttnConfig, w, device, heads, kv_names, *, uk_pack=None, nb: int = 1, dlat: int = 0,
                 drp: int | None = None, absorbed: bool | None = False, score_scale: float = 1.0):
        import numpy as np

        self.cfg = cfg
        self.device = torch.device(device)
        self.heads = list(heads)
        H = len(self.heads)
        d_h, dr = cfg.d_h, cfg.d_h_rope
        get = lambda n: np.asarray(w[n], dtype=np.float64)  # noqa: E731
        w_dq, w_uq, w_qr, w_kr = get("w_dq"), get("w_uq"), get("w_qr"), get("w_kr")
        self.kv_names = list(kv_names)
        kvs = [get(n) for n in self.kv_names]
        self.n_q, self.n_kv, self.n_kr = w_dq.shape[1], sum(k.shape[1] for k in kvs), w_kr.shape[1]
        self.kv_cols = {}
        c = 0
        for n, k in zip(self.kv_names, kvs):
            self.kv_cols[n] = (c, c + k.shape[1])
            c += k.shape[1]
        self.d_cq = w_dq.shape[1]
        self.w_down, self.w_down_slabs = self._pack(np.concatenate([w_dq, *kvs, w_kr], axis=1))
        uq = w_uq.reshape(self.d_cq, cfg.h, d_h)[:, self.heads]
        qr = w_qr.reshape(self.d_cq, cfg.h, dr)[:, self.heads].reshape(self.d_cq, H * dr)
        if absorbed is None:
            absorbed = uk_pack is not None and nb * dlat <= d_h
        self.absorbed = bool(absorbed)
        if self.absorbed:
            uk = np.asarray(uk_pack, dtype=np.float64).reshape(H, d_h, nb, dlat)  # [H, d_h, NB*DLAT] pack
            wq = np.einsum("khp,hpbc->kbhc", uq, uk).reshape(self.d_cq, nb * H * dlat)
            self.q_shape = (nb, H, dlat)
            self.q_scale = self.r_scale = float(score_scale)
        else:
            wq = uq.reshape(self.d_cq, H * d_h)
            self.q_shape = (H, d_h)
            self.q_scale = self.r_scale = 1.0
        self.nq = wq.shape[1]
        self.w_query, self.w_query_slabs = self._pack(np.concatenate([wq, qr], axis=1))
        self.H, self.dr = H, dr
        self.drp = drp if drp is not None else dr
        sf = calib_factors(cfg)
        self.alpha_q, self.alpha_kv = float(sf.alpha_q), float(sf.alpha_kv)
        self._bufs: dict = {}
        self._w2 = None

    def _pack(self, m):
        """bf16 [K, N] (cuBLAS paths) and its slab pack for K-1 (``ops.slab_pack``)."""
        plain = torch.as_tensor(m, dtype=torch.float32).to(device=self.device, dtype=torch.bfloat16).contiguous()
        return plain, ops.slab_pack(plain)

    def buffers(self, M: int) -> dict:
        b = self._bufs.get(M)
        if b is None:
            f32 = dict(dtype=torch.float32, device=self.device)
            b = {"c_q_raw": torch.empty((M, self.n_q), **f32), "kv_raw": torch.empty((M, self.n_kv), **f32),
                 "kr_raw": torch.empty((M, self.n_kr), **f32),
                 "ssq": torch.empty((-(-self.n_q // 64), M), **f32),
                 "q": torch.empty((M,) + self.q_shape, dtype=torch.bfloat16, device=self.device),
                 "r": torch.zeros((M, self.H, self.drp), dtype=torch.bfloat16, device=self.device)}
            self._bufs[M] = b
        return b

    def down(self, hidden: torch.Tensor):
        """K-1 down for hidden [M <= 16, d] fp32 (device): (c_q_raw, kv_raw [M, n_kv], kr_raw [M, dr])
        fp32 plus the query rmsnorm statistics, kept for ``query``."""
        M = hidden.shape[0]
        if M > 16:
            raise ShapeMismatchError("KernelProjector.down: at most 16 rows per call (use project)")
        b = self.buffers(M)
        ops.proj_down(hidden, self.w_down_slabs, self.n_q, self.n_kv, self.n_kr, b["c_q_raw"], b["kv_raw"], b["kr_raw"],
                      b["ssq"])
        return b["kv_raw"], b["kr_raw"]

    def query(self, M: int, pos: torch.Tensor, pos_delta: int = 0):
        """K-1 query for the rows of the last ``down``: (q [M, ...] bf16, q_rope [M, H, drp] bf16)
        with the rope at pos + pos_delta."""
        b = self.buffers(M)
        ops.proj_query(b["c_q_raw"], b["ssq"], self.alpha_q, self.w_query_slabs, self.nq, self.H, self.dr, pos, b["q"],
                       b["r"], q_scale=self.q_scale, r_scale=self.r_scale, pos_delta=pos_delta)
        return b["q"], b["r"]

    def project(self, hidden: torch.Tensor, pos: torch.Tensor):
        """hidden [M, d] fp32, pos [M] int32 -> (kv_raw [M, n_kv] fp32, kr_raw [M, dr] fp32, q [M, ...]
        bf16 (q_nope [M, H, d_h] or q~ [M, NB, H, DLAT]), q_rope [M, H, drp] bf16 (rope applied;
        scaled by tau*log2e when absorbed)), in chunks of 16 rows (the rmsnorm statistics of a
        chunk travel from the down to the query kernel)."""
        hidden = hidden.to(device=self.device, dtype=torch.float32).contiguous()
        pos = pos.to(device=self.device, dtype=torch.int32).contiguous()
        M = hidden.shape[0]
        if M <= 16:
            kv, kr = self.down(hidden)
            q, r = self.query(M, pos)
            return kv, kr, q, r
        outs = [self.project(hidden[m0:m0 + 16], pos[m0:m0 + 16]) for m0 in range(0, M, 16)]
        return tuple(torch.cat([o[i] for o in outs]) for i in range(4))

    def project_gemm(self, hidden: torch.Tensor, pos0: int, drq: int | None = None, rope_scale: float | None = None):
        """``project`` for the n rows of a prefill at positions pos0 .. pos0+n-1: the same packed
        bf16 weights through cuBLAS bf16 GEMMs (real GEMMs at n rows, where a weight stream per 16
        rows would not pay), the activations as bf16 hi + lo (``ops.rows_split``, with the query
        rmsnorm) like K-1's operands, and ``ops.query_epilogue`` for the scaling and rope. Returns
        (kv_raw, kr_raw, q [n, ...] bf16, q_rope [n, H, drq] bf16); ``rope_scale`` overrides the
        rotary query's scale (the prefill kernel takes it pre-scaled by tau*log2e)."""
        hidden = hidden.to(device=self.device, dtype=torch.float32).contiguous()
        n = hidden.shape[0]
        if self._w2 is None:  # [W; W] for the one-GEMM hi + lo product
            self._w2 = (torch.cat([self.w_down, self.w_down]), torch.cat([self.w_query, self.w_query]))
        y = _gemm2(ops.rows_split(hidden, hidden.shape[1], stacked=True), self._w2[0])
        n_q, n_kv = self.n_q, self.n_kv
        kv_raw = y[:, n_q:n_q + n_kv].contiguous()
        kr_raw = y[:, n_q + n_kv:n_q + n_kv + self.n_kr].contiguous()
        q = _gemm2(ops.rows_split(y, n_q, norm=True, alpha=self.alpha_q, stacked=True), self._w2[1])
        r_scale = self.r_scale if rope_scale is None else rope_scale
        qx, qr = ops.query_epilogue(q, self.nq, self.H, self.dr, drq or self.drp, pos0, self.q_scale, r_scale)
        return kv_raw, kr_raw, qx.reshape((n,) + self.q_shape), qr

    def kv_slice(self, kv_raw: torch.Tensor, names) -> torch.Tensor:
        """The raw columns of the given down-projections (contiguous, in kv_names order)."""
        lo, hi = self.kv_cols[names[0]][0], self.kv_cols[names[-1]][1]
        return kv_raw[:, lo:hi].contiguous()
