"""Decode steps fed from and drained to pinned host memory, with the copies off the critical path.

The reference steps one token at a time from host arrays (``decode.py:341-348`` decode_step
-> ``decode.py:129-150`` append + ``decode.py:217-305`` attend/reduce). A serving loop on the
B200 keeps several micro-batches in flight instead: while micro-batch k runs K0..K3, the next
micro-batch's inputs are uploaded and the previous one's output is downloaded.

``MicroBatchLoop`` does that over a list of ``DecodeEngine`` objects (one paged cache each).
Per step of micro-batch k:

* upload stream: ONE host->device copy of k's pinned staging buffer ``[rows | q_nope | q_rope]``
  (the new token's cache rows and its queries), after k's previous step has consumed it, then
  K0 with ``advance=1`` (writes the token row and bumps ``seqlens``: no separate length
  update) -- both under the other micro-batch's kernels;
* compute stream: K1 -> K2 -> K3 into the engine's output buffer;
* download stream: ONE device->host copy of the fp32 output into k's pinned result buffer.

Host contract: ``wait(k)`` returns when k's last submitted step is fully done; after it,
``host_output(k)`` holds that step's result and ``host_inputs(k)`` may be refilled for the next
``submit(k)``. (Re-submitting k without ``wait`` re-sends whatever the staging buffer holds.)
"""

from __future__ import annotations

import math

import torch

from . import ops
from .errors import ConfigError

__all__ = ["MicroBatchLoop"]


class _Slot:
    def __init__(self, eng):
        c = eng.cache
        lay = eng.layout
        B, hl, dh = c.batch, len(eng.heads), eng.cfg.d_h
        self.eng = eng
        self.shapes = [(B, lay.width), (B, hl, dh), (B, hl, lay.drp)]
        self.offsets, n = [], 0
        for s in self.shapes:  # each view starts 256-byte aligned
            self.offsets.append(n)
            n += -(-math.prod(s) // 128) * 128
        self.h_in = torch.zeros(n, dtype=torch.bfloat16).pin_memory()
        self.d_in = torch.empty(n, dtype=torch.bfloat16, device=eng.device)
        self.h_out = torch.empty((B, hl, dh), dtype=torch.float32).pin_memory()
        self.up_done = torch.cuda.Event()
        self.step_done = torch.cuda.Event()
        self.down_done = torch.cuda.Event()

    def views(self, flat):
        return [flat[o:o + math.prod(s)].view(s) for s, o in zip(self.shapes, self.offsets)]


class MicroBatchLoop:
    """Micro-batches of one device stepped in turn with overlapped host<->device copies."""

    def __init__(self, engines, reducer=None, graphs=False):
        """reducer: collective.PeerAllReduce of the engines' TP group (B*h*d_h values): every step
        then runs ``decode_attention_tp`` (the sum over the group fused into K3), so the result
        downloaded is the full TP output. All ranks must submit the same micro-batch sequence.
        graphs: each micro-batch's K1..K3 call (its inputs are the slot's fixed device staging
        views, its output the engine's buffer, the lengths advance on the device) is captured
        once, after one eager step, and replayed -- one launch instead of the per-kernel host
        calls. The copies and K0 stay eager on their streams (the cross-step events)."""
        if not engines:
            raise ConfigError("MicroBatchLoop needs at least one engine")
        dev = engines[0].device
        if any(e.device != dev for e in engines):
            raise ConfigError("MicroBatchLoop: all micro-batches must live on one device")
        self.device = dev
        self.slots = [_Slot(e) for e in engines]
        self.up = torch.cuda.Stream(device=dev)
        self.down = torch.cuda.Stream(device=dev)
        self.reducer = reducer
        self.graphs = graphs
        self._graph = [None] * len(engines)
        self._eager_steps = [0] * len(engines)

    def __len__(self) -> int:
        return len(self.slots)

    def host_inputs(self, k: int):
        """Pinned (rows [B, W], q_nope [B, h_local, d_h], q_rope [B, h_local, drp]) bf16 views."""
        return tuple(self.slots[k].views(self.slots[k].h_in))

    def host_output(self, k: int) -> torch.Tensor:
        return self.slots[k].h_out

    def bytes_per_step(self, k: int = 0) -> tuple[int, int]:
        s = self.slots[k]
        return s.h_in.numel() * s.h_in.element_size(), s.h_out.numel() * s.h_out.element_size()

    def submit(self, k: int) -> None:
        """Enqueue one step of micro-batch k (upload, K0..K3, download); returns immediately."""
        s = self.slots[k]
        eng = s.eng
        c = eng.cache
        c.reserve_token()
        main = torch.cuda.current_stream(self.device)
        self.up.wait_event(s.step_done)  # k's previous step has read its staging buffer
        rows, qn, qr = s.views(s.d_in)
        with torch.cuda.stream(self.up):
            s.d_in.copy_(s.h_in, non_blocking=True)
            # K0 on the upload stream too: it runs under the other micro-batch's kernels
            ops.cache_append(rows, c.block_table, c.seqlens, c.pool, c.page_size, advance=True)
            s.up_done.record(self.up)
        main.wait_event(s.up_done)
        main.wait_event(s.down_done)  # the output buffer has been drained
        if self._graph[k] is not None:
            self._graph[k].replay()
            out = eng.out
        else:
            out = self._attention(eng, qn, qr)
            self._eager_steps[k] += 1
            if self.graphs and self._eager_steps[k] == 1:
                self._capture(k, eng, qn, qr, main)
        s.step_done.record(main)
        self.down.wait_event(s.step_done)
        with torch.cuda.stream(self.down):
            s.h_out.copy_(out, non_blocking=True)
            s.down_done.record(self.down)

    def _attention(self, eng, qn, qr):
        if self.reducer is not None:
            return eng.decode_attention_tp(qn, qr, self.reducer, out=eng.out)
        return eng.decode_attention(qn, qr, out=eng.out)

    def _capture(self, k, eng, qn, qr, main):
        """Capture micro-batch k's K1..K3 (after its first eager step set up the tensor maps and
        workspace). Capture does not execute: the step just run is not repeated."""
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(main)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self._attention(eng, qn, qr)
        main.wait_stream(side)
        self._graph[k] = g

    def wait(self, k: int) -> torch.Tensor:
        self.slots[k].down_done.synchronize()
        return self.slots[k].h_out

    def join(self) -> None:
        """Make the current stream wait for every outstanding download (no host sync)."""
        main = torch.cuda.current_stream(self.device)
        for s in self.slots:
            main.wait_event(s.down_done)

    def start(self) -> None:
        """Order the copy streams after work already queued on the current stream."""
        main = torch.cuda.current_stream(self.device)
        self.up.wait_stream(main)
        self.down.wait_stream(main)
