"""Seeded weights and synthetic inputs, bit-compatible with the reference kit.

``Rng`` is a label-splittable counter-based (Philox) stream whose key is a
blake2b-128 digest of the seed and label path, so the same (seed, labels) draw
the same numbers as attnkit/tensors.py:20-53. ``build_weights`` draws every
matrix of a variant under ``rng.split(name)`` with the shapes of
attnkit/weights.py:45-113 (latent family and gqa are what the decode path uses).
This is host plumbing: it produces float64 numpy arrays that the GPU path packs
to bf16 once (see ``decode.pack_weights``).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

from .config import AttnConfig
from .errors import ConfigError, NumericError


def _philox_key(seed: int, path: tuple[str, ...]) -> int:
    h = hashlib.blake2b(digest_size=16)
    h.update(str(int(seed)).encode())
    for label in path:
        h.update(b"/")
        h.update(label.encode())
    return int.from_bytes(h.digest(), "little")


class Rng:
    """Philox stream keyed by (seed, label path); ``split`` derives a child by label."""

    def __init__(self, seed: int, _path: tuple[str, ...] = ()):
        self.seed = int(seed)
        self._path = _path
        self._gen = np.random.Generator(np.random.Philox(key=_philox_key(self.seed, _path)))

    def split(self, label) -> "Rng":
        return Rng(self.seed, self._path + (str(label),))

    def normal(self, shape, sigma: float = 1.0) -> np.ndarray:
        if sigma == 0.0:
            return np.zeros(shape, dtype=np.float64)
        return sigma * self._gen.standard_normal(size=shape, dtype=np.float64)

    def integers(self, low: int, high: int) -> int:
        return int(self._gen.integers(low, high))


@dataclass
class WeightSet:
    variant: str
    tensors: dict[str, np.ndarray] = field(default_factory=dict)

    def __getitem__(self, name: str) -> np.ndarray:
        try:
            return self.tensors[name]
        except KeyError:
            raise ConfigError(f"weight set for {self.variant!r} has no tensor {name!r}") from None

    def __contains__(self, name: str) -> bool:
        return name in self.tensors

    def element_count(self) -> int:
        return sum(t.size for t in self.tensors.values())


def weight_shapes(cfg: AttnConfig) -> dict[str, tuple[int, int]]:
    """Matrix shapes per weight name (attnkit/weights.py:45-99, latent + gqa branches)."""
    h, d, d_h = cfg.h, cfg.d, cfg.d_h
    v = cfg.variant
    if v in ("mqa", "gqa"):
        shapes = {"w_q": (d, h * d_h), "w_k": (d, cfg.g * d_h), "w_v": (d, cfg.g * d_h)}
    elif v == "mha":
        shapes = {"w_q": (d, h * d_h), "w_k": (d, h * d_h), "w_v": (d, h * d_h)}
    elif v in ("mla", "gla", "mlra"):
        shapes = {
            "w_dq": (d, cfg.d_cq),
            "w_uq": (cfg.d_cq, h * d_h),
            "w_qr": (cfg.d_cq, h * cfg.d_h_rope),
            "w_kr": (d, cfg.d_h_rope),
        }
        if grouped_latents(cfg):
            r = h // cfg.g
            dg = cfg.group_latent_dim
            for j in range(cfg.g):
                shapes[f"w_dkv_{j}"] = (d, dg)
                shapes[f"w_uk_{j}"] = (dg, r * d_h)
                shapes[f"w_uv_{j}"] = (dg, r * d_h)
        else:
            shapes["w_dkv"] = (d, cfg.d_c)
            shapes["w_uk"] = (cfg.d_c, h * d_h)
            shapes["w_uv"] = (cfg.d_c, h * d_h)
    else:
        raise ConfigError(f"no weight table for variant {v!r} on the decode path")
    if cfg.gated:
        shapes["w_g"] = (d, cfg.out_flat_dim)
    shapes["w_o"] = (cfg.out_flat_dim, d)
    return shapes


def grouped_latents(cfg: AttnConfig) -> bool:
    return cfg.variant == "gla" or (cfg.variant == "mlra" and cfg.branches == 2)


def gaussian_init(shape, sigma: float, rng: Rng) -> np.ndarray:
    if sigma < 0:
        raise NumericError(f"gaussian_init: negative sigma {sigma}")
    return rng.normal(shape, sigma)


def build_weights(cfg: AttnConfig, sigma: float, rng: Rng, out_sigma: float | None = None) -> WeightSet:
    tensors = {}
    for name, shape in weight_shapes(cfg).items():
        s = sigma if name != "w_o" or out_sigma is None else out_sigma
        tensors[name] = gaussian_init(shape, s, rng.split(name))
    return WeightSet(cfg.variant, tensors)
