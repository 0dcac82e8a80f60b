"""Calibration factors and the analytic traffic/FLOP formulas the bench reports against.

``calib_factors`` follows attnkit/latent.py:41-69 (alpha_q, alpha_kv, alpha_attn; alpha_attn =
1/sqrt(branches) for mlra). ``per_device_load`` / ``decode_flops_per_device`` follow
attnkit/costs.py:70-127 and define the ALGORITHMIC bytes and FLOPs used for roofline
fractions: bytes = sum over sequences of n * per_device_load * d_h * 2 (bf16, costs.py:18).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .config import LATENT_VARIANTS, TP_DEGREES, AttnConfig
from .errors import ConfigError

CACHE_BYTES_PER_ELEMENT = 2


@dataclass(frozen=True)
class ScaleFactors:
    alpha_q: float
    alpha_kv: float
    alpha_attn: float


def calib_factors_squared(cfg: AttnConfig) -> tuple[Fraction, Fraction, Fraction]:
    if not cfg.scaling:
        return Fraction(1), Fraction(1), Fraction(1)
    if cfg.variant == "mla":
        return Fraction(cfg.d, cfg.d_cq), Fraction(cfg.d, cfg.d_c), Fraction(1)
    if cfg.variant == "gla":
        return Fraction(cfg.d, cfg.d_cq), Fraction(cfg.g * cfg.d, cfg.d_c), Fraction(1)
    if cfg.variant == "mlra":
        return Fraction(cfg.d, cfg.d_cq), Fraction(4 * cfg.d, cfg.d_c), Fraction(1, cfg.branches)
    raise ConfigError(f"no calibration factors for variant {cfg.variant!r}")


def calib_factors(cfg: AttnConfig) -> ScaleFactors:
    if cfg.variant not in LATENT_VARIANTS:
        return ScaleFactors(1.0, 1.0, 1.0)
    q2, kv2, a2 = calib_factors_squared(cfg)
    return ScaleFactors(float(q2) ** 0.5, float(kv2) ** 0.5, float(a2) ** 0.5)


def fraction_str(x: Fraction) -> str:
    """Exact decimal string when the denominator has only factors 2 and 5 ("1.5"), else "p/q"
    (the ledger/report convention of attnkit/costs.py:351-370)."""
    import decimal

    den = x.denominator
    for f in (2, 5):
        while den % f == 0:
            den //= f
    if den != 1:
        return f"{x.numerator}/{x.denominator}"
    with decimal.localcontext() as ctx:
        ctx.prec = 60
        d = (decimal.Decimal(x.numerator) / decimal.Decimal(x.denominator)).normalize()
    s = format(d, "f")
    return s


def _check_phi(phi: int) -> None:
    if phi not in TP_DEGREES:
        raise ConfigError(f"unsupported TP degree {phi}; supported: {TP_DEGREES}")


def kv_cache_per_token(cfg: AttnConfig) -> Fraction:
    """Cached elements per token, in d_h units (costs.py:52-67, served variants)."""
    if cfg.variant in ("mqa", "gqa"):
        return Fraction(2 * cfg.g * cfg.d_h, cfg.d_h)
    if cfg.variant == "mha":
        return Fraction(2 * cfg.h)
    return Fraction(cfg.d_c + cfg.d_h_rope, cfg.d_h)


def per_device_load(cfg: AttnConfig, phi: int) -> Fraction:
    """Cache elements one device reads per past token per step, in d_h units (costs.py:70-102)."""
    _check_phi(phi)
    v = cfg.variant
    if v == "mha":
        return Fraction(2 * cfg.h, phi)
    if v == "mqa":
        return Fraction(2)
    if v == "gqa":
        return Fraction(2 * cfg.g, min(phi, cfg.g))
    if v == "mla":
        return Fraction(cfg.d_c + cfg.d_h_rope, cfg.d_h)
    if v == "gla":
        return Fraction(cfg.d_c, min(phi, cfg.g) * cfg.d_h) + Fraction(cfg.d_h_rope, cfg.d_h)
    if v == "mlra":
        return Fraction(cfg.d_c, min(phi, 4) * cfg.d_h) + Fraction(cfg.d_h_rope, cfg.d_h)
    raise ConfigError(f"no loading rule for {v!r}")


def decode_flops_per_device(cfg: AttnConfig, phi: int, n: int) -> Fraction:
    """Attention FLOPs per device per decode step over an n-token cache (costs.py:105-127)."""
    _check_phi(phi)
    v = cfg.variant
    heads = Fraction(cfg.h, phi)
    if v in ("mha", "mqa", "gqa", "gta"):
        return heads * 4 * n * cfg.d_h
    if v == "mla":
        return heads * (4 * n * cfg.d_c + 2 * n * cfg.d_h_rope)
    if v == "gla":
        return heads * (4 * n * Fraction(cfg.d_c, cfg.g) + 2 * n * cfg.d_h_rope)
    pairs = Fraction(cfg.branches * cfg.h, phi)
    return pairs * (4 * n * Fraction(cfg.d_c, 4) + 2 * n * cfg.d_h_rope)


def algorithmic_bytes(cfg: AttnConfig, phi: int, seqlens) -> int:
    """Per-device cache bytes one decode step must read: sum_n n * load * d_h * 2."""
    load = per_device_load(cfg, phi) * cfg.d_h * CACHE_BYTES_PER_ELEMENT
    total = sum(int(n) for n in seqlens) * load
    if total.denominator != 1:
        raise ConfigError("per-device load is not a whole number of bytes per token")
    return int(total)
