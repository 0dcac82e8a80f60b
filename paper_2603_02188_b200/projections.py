"""Pre-attention projections on the GPU (torch/cuBLAS, fp32): the rows a decode step
appends and the queries it attends with.

Restates attnkit/latent.py:129-159 (latent_projections) and attnkit/zoo.py:53-58 (gqa)
for the drop-in ``absorbed_decode_step``. This is plumbing around the hot path (SURVEY.md
section 8(f) row 1 lists its fusion into a kernel as the next step), not part of the
measured decode-attention step.
"""

from __future__ import annotations

import torch

from .config import AttnConfig
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
