"""Paged bf16 latent KV cache in device memory (replaces attnkit/cache.py:24-84).

Physical layout (what the K2 kernel's TMA descriptors expect):

* a pool ``[num_pages * page_size, W]`` bf16, one row per token slot, where a row is
  ``[unit 0 latent | unit 1 latent | ... | rope]``; every latent unit (an MLRA block
  ``latent_b{k}`` or the whole MLA ``latent``) is zero-padded to ``dlp`` columns (64 or a
  multiple of 128) and the rotary key to ``drp`` (a multiple of 16). Zero columns change
  neither the logits (the queries are padded with zeros too) nor the value mixture (the
  padded W^UV rows are zero), so any reference config can run on the same kernels;
* a block table ``[B, max_pages]`` int32 of page ids and ``seqlens [B]`` int32.

``PagedCache`` is the batched serving object. ``PagedLatentCache`` wraps one sequence of
it behind the reference ``KvCache`` protocol (``n``, ``pos_offset``, ``row_shapes``,
``streams``, ``reads``, ``row_elements``, ``append``, ``read``, ``peek``, ``row``,
``fingerprint``) so it drops into attnkit-style callers. ``read``/``peek`` are debug
device-to-host copies; the ``reads`` counter stays analytic (elements a decode step
touches), exactly like ``KvCache.read`` charges them (cache.py:59-66).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ConfigError, ShapeMismatchError


def _pad_latent(width: int) -> int:
    if width <= 64:
        return 64
    return -(-width // 128) * 128


def _pad_rope(width: int) -> int:
    p = max(16, -(-width // 16) * 16)
    if p > 64:
        raise ConfigError(f"rotary key width {width} exceeds the kernel's 64-column rope tile")
    return p


@dataclass(frozen=True)
class RowLayout:
    """Token-row layout of the pool: latent units (in order) + shared rotary key."""

    units: tuple  # stream names, e.g. ("latent_b0", ..., "latent_b3") or ("latent",)
    dl: int       # logical latent width per unit
    dr: int       # logical rotary width

    @property
    def dlp(self) -> int:
        return _pad_latent(self.dl)

    @property
    def drp(self) -> int:
        return _pad_rope(self.dr)

    @property
    def nb(self) -> int:
        return len(self.units)

    @property
    def width(self) -> int:
        return self.nb * self.dlp + self.drp

    @property
    def geometry(self) -> tuple[int, int]:
        return ops.latent_geometry(self.dlp)

    def row_shapes(self) -> dict:
        shapes = {u: (self.dl,) for u in self.units}
        shapes["rope"] = (self.dr,)
        return shapes

    def column(self, name: str) -> slice:
        if name == "rope":
            o = self.nb * self.dlp
            return slice(o, o + self.dr)
        i = self.units.index(name)
        return slice(i * self.dlp, i * self.dlp + self.dl)

    def extract(self, name: str, rows: torch.Tensor) -> torch.Tensor:
        """[..., W] pool rows -> [..., *row_shape] of one stream."""
        return rows[..., self.column(name)]

    def pack_rows(self, rows: dict, device=None) -> torch.Tensor:
        """{stream: [..., width]} (numpy or torch, any float) -> [..., W] bf16 padded rows."""
        first = next(iter(rows.values()))
        lead = tuple(first.shape[:-1])
        out = torch.zeros(lead + (self.width,), dtype=torch.float32, device=device)
        for name in list(self.units) + ["rope"]:
            v = rows[name]
            v = torch.as_tensor(np.asarray(v) if not torch.is_tensor(v) else v, dtype=torch.float32, device=device)
            out[..., self.column(name)] = v
        return out.to(torch.bfloat16)


@dataclass(frozen=True)
class GqaLayout:
    """Token-row layout of a GQA pool (the comparison variant, attnkit/zoo.py:47-58 streams
    ``k`` and ``v`` of shape (g, d_h), cache.py:105-144): ``[K_0 | ... | K_{g-1} | V_0 | ... |
    V_{g-1}]``, each KV head zero-padded to ``dhp`` in {64, 128} columns (zero key columns
    leave the logits unchanged, zero value columns are sliced off the output)."""

    g: int   # KV heads held by this device
    dh: int  # head width

    @property
    def dhp(self) -> int:
        if self.dh > 128:
            raise ConfigError(f"gqa head width {self.dh} exceeds the kernel's 128-column sub-block")
        return 64 if self.dh <= 64 else 128

    @property
    def units(self) -> tuple:
        return ("k", "v")

    @property
    def width(self) -> int:
        return 2 * self.g * self.dhp

    def row_shapes(self) -> dict:
        return {"k": (self.g, self.dh), "v": (self.g, self.dh)}

    def extract(self, name: str, rows: torch.Tensor) -> torch.Tensor:
        if name not in ("k", "v"):
            raise ConfigError(f"gqa cache has no stream {name!r}")
        o = 0 if name == "k" else self.g * self.dhp
        part = rows[..., o:o + self.g * self.dhp]
        return part.reshape(*part.shape[:-1], self.g, self.dhp)[..., :self.dh]

    def pack_rows(self, rows: dict, device=None) -> torch.Tensor:
        """{"k": [..., g, d_h], "v": [..., g, d_h]} -> [..., W] bf16 padded rows."""
        k, v = (torch.as_tensor(np.asarray(rows[n]) if not torch.is_tensor(rows[n]) else rows[n],
                                dtype=torch.float32, device=device) for n in ("k", "v"))
        lead = tuple(k.shape[:-2])
        out = torch.zeros(lead + (2, self.g, self.dhp), dtype=torch.float32, device=device)
        out[..., 0, :, :self.dh] = k
        out[..., 1, :, :self.dh] = v
        return out.reshape(lead + (self.width,)).to(torch.bfloat16)


class PagedCache:
    """Batched paged latent cache on one device.

    ``B`` sequences, each with up to ``max_tokens`` tokens, pages of ``page_size`` token slots.
    Pages are assigned from a flat pool; ``page_order`` may permute them (tests use a random
    permutation to exercise non-contiguous page tables).
    """

    def __init__(self, layout: RowLayout, batch: int, max_tokens: int, page_size: int = 128, device=None,
                 page_order: torch.Tensor | None = None):
        if page_size % 64:
            raise ConfigError(f"page_size {page_size} must be a multiple of 64 tokens")
        self.layout = layout
        self.batch = int(batch)
        self.page_size = int(page_size)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.max_pages = max(1, -(-int(max_tokens) // page_size))
        self.num_pages = self.batch * self.max_pages
        self.pool = torch.zeros((self.num_pages * page_size, layout.width), dtype=torch.bfloat16, device=self.device)
        order = torch.arange(self.num_pages, dtype=torch.int32) if page_order is None else page_order.to(torch.int32)
        self.block_table = order[: self.batch * self.max_pages].reshape(self.batch, self.max_pages).to(self.device)
        self.seqlens = torch.zeros(self.batch, dtype=torch.int32, device=self.device)
        self._host_lens = [0] * self.batch

    @property
    def capacity(self) -> int:
        return self.max_pages * self.page_size

    def lengths(self) -> list[int]:
        return list(self._host_lens)

    def reserve_token(self) -> None:
        """Host bookkeeping for one appended token per sequence (capacity check first)."""
        if max(self._host_lens) >= self.capacity:
            raise ConfigError(f"cache full: capacity {self.capacity} tokens per sequence")
        self._host_lens = [n + 1 for n in self._host_lens]

    def append(self, rows: torch.Tensor) -> None:
        """K0: write one new token row per sequence ([B, W] bf16, device) at its current end."""
        if rows.shape != (self.batch, self.layout.width):
            raise ShapeMismatchError(f"append: rows {tuple(rows.shape)} != {(self.batch, self.layout.width)}")
        self.reserve_token()
        ops.cache_append(rows.contiguous(), self.block_table, self.seqlens, self.pool, self.page_size, advance=True)

    def append_latent(self, kv_raw: torch.Tensor, kr_raw: torch.Tensor, rope_pos, *, branches: int, block0: int,
                      nblocks: int, alpha_kv: float, rope_base: float = 10000.0, norm_groups: int = 1) -> None:
        """Fused K0 for one new token per sequence: kv_raw [B, d_c] / kr_raw [B, dr] fp32 raw
        projections, rope_pos [B] absolute positions (host list or int32 device tensor)."""
        lay = self.layout
        self.reserve_token()
        pos = rope_pos if torch.is_tensor(rope_pos) else torch.tensor(list(rope_pos), dtype=torch.int32)
        ops.cache_append_latent(kv_raw.float().contiguous(), kr_raw.float().contiguous(),
                                pos.to(device=self.device, dtype=torch.int32), self.seqlens, self.block_table,
                                self.pool, self.page_size, branches=branches, block0=block0, nblocks=nblocks,
                                dlp=lay.dlp, drp=lay.drp, alpha_kv=alpha_kv, rope_base=rope_base,
                                norm_groups=norm_groups, advance=True)

    def fill(self, rows: torch.Tensor, lengths) -> None:
        """Bulk prefill: rows [B, n_max, W] bf16 (device); sequence s keeps its first lengths[s]."""
        lengths = [int(x) for x in lengths]
        if max(lengths) > self.capacity:
            raise ConfigError(f"fill: {max(lengths)} tokens exceed capacity {self.capacity}")
        ps = self.page_size
        bt = self.block_table.long()
        for s, n in enumerate(lengths):
            if n == 0:
                continue
            tok = torch.arange(n, device=self.device)
            slots = bt[s, tok // ps] * ps + tok % ps
            self.pool[slots] = rows[s, :n].to(torch.bfloat16)
        self.seqlens.copy_(torch.tensor(lengths, dtype=torch.int32))
        self._host_lens = lengths

    def token_slots(self, s: int) -> torch.Tensor:
        n = self._host_lens[s]
        tok = torch.arange(n, device=self.device)
        return self.block_table[s].long()[tok // self.page_size] * self.page_size + tok % self.page_size

    def stream(self, s: int, name: str) -> torch.Tensor:
        """Device view (copy) of one stream of sequence s: [n, *row_shape] bf16."""
        return self.layout.extract(name, self.pool[self.token_slots(s)])


class PagedLatentCache:
    """One sequence behind the reference KvCache protocol (attnkit/cache.py:24-84)."""

    def __init__(self, variant: str, layout: RowLayout, pos_offset: int = 0, device=None, page_size: int = 128,
                 initial_tokens: int = 1024):
        self.variant = variant
        self.layout = layout
        self.pos_offset = int(pos_offset)
        self.reads = 0
        self._page_size = page_size
        self._device = device
        self.paged = PagedCache(layout, 1, max(initial_tokens, page_size), page_size, device)

    # -- protocol -----------------------------------------------------------------
    @property
    def n(self) -> int:
        return self.paged.lengths()[0]

    @property
    def row_shapes(self) -> dict:
        return self.layout.row_shapes()

    @property
    def streams(self) -> tuple:
        return tuple(self.row_shapes)

    def row_elements(self) -> int:
        return sum(int(np.prod(s)) for s in self.row_shapes.values())

    def append(self, rows: dict) -> None:
        """Append one token (cache.py:44-57): exactly the owned streams, each of its row shape."""
        if set(rows) != set(self.row_shapes):
            raise ShapeMismatchError(
                f"cache append: got streams {sorted(rows)}, expected {sorted(self.row_shapes)}"
            )
        for name, row in rows.items():
            shape = tuple(np.shape(row))
            if shape != self.row_shapes[name]:
                raise ShapeMismatchError(
                    f"cache append: stream {name!r} row shape {shape}, expected {self.row_shapes[name]}"
                )
        self.append_packed(self.layout.pack_rows(rows, device=self.paged.device)[None])

    def append_packed(self, row: torch.Tensor) -> None:
        """Append an already packed [1, W] bf16 device row (the decode fast path)."""
        if self.n >= self.paged.capacity:
            self._grow()
        self.paged.append(row)

    def append_latent(self, kv_raw: torch.Tensor, kr_raw: torch.Tensor, rope_pos: int, *, branches: int,
                      block0: int, nblocks: int, alpha_kv: float, norm_groups: int = 1) -> None:
        """Fused write side (K0): rmsnorm*alpha_kv of the raw down-projection [1, d_c], rope of the
        raw rotary key [1, dr] at rope_pos, owned blocks + key appended as one row."""
        if self.n >= self.paged.capacity:
            self._grow()
        self.paged.append_latent(kv_raw, kr_raw, [rope_pos], branches=branches, block0=block0, nblocks=nblocks,
                                 alpha_kv=alpha_kv, norm_groups=norm_groups)

    def read(self, name: str) -> np.ndarray:
        """Debug copy of one stream as float64 [n, width], charging n*width reads."""
        out = self.peek(name)
        self.reads += out.size
        return out

    def peek(self, name: str) -> np.ndarray:
        if name not in self.row_shapes:
            raise ConfigError(f"cache read: no stream {name!r}")
        if self.n == 0:
            raise ConfigError(f"cache read: stream {name!r} is empty")
        return self.paged.stream(0, name).float().cpu().numpy().astype(np.float64)

    def row(self, name: str, t: int) -> np.ndarray:
        """Stored row of token t (frozen copy: writing to it raises, as in cache.py:72-74)."""
        if not 0 <= t < self.n:
            raise IndexError(t)
        slot = self.paged.token_slots(0)[t]
        out = self.layout.extract(name, self.paged.pool[slot]).float().cpu().numpy().astype(np.float64)
        out.setflags(write=False)
        return out

    def fingerprint(self, upto: int | None = None) -> str:
        upto = self.n if upto is None else upto
        h = hashlib.sha256()
        for name in sorted(self.row_shapes):
            h.update(name.encode())
            if upto:
                h.update(np.ascontiguousarray(self.peek(name)[:upto]).tobytes())
        return h.hexdigest()

    # -- internals ----------------------------------------------------------------
    def _grow(self) -> None:
        old = self.paged
        new = PagedCache(self.layout, 1, 2 * old.capacity, self._page_size, old.device)
        n = self.n
        if n:
            new.pool[:n] = old.pool[old.token_slots(0)]  # identity page order: token t -> slot t
        new.seqlens.fill_(n)
        new._host_lens = [n]
        self.paged = new
