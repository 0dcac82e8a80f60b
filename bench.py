"""Benchmark: MLRA-4 decode attention on B200 (BASELINE.json metric / configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1  -> configs[1]: 2.9B MLRA-4 layer (h=24, d_h=128, d_c=512, d_h^R=64), batch 16, 32K
          context, all four branches on one GPU (TP1). The same JSON line also carries the
          headline per-GPU TP4 number (one TP4 rank's share of the same batch) and the MLA
          comparison at the same shapes (TP4 heads-sharded rank, and TP1).
N = 2/4 -> TP2 / TP4 over the same batch of 16 (torchrun, NCCL all-reduce of the branch
          outputs); N = 8 -> 2 x TP4 over a batch of 32 (16 per TP group).

A "step" is one decode-attention step for the whole batch: K1 absorb -> K2 split-KV
flash-decode -> K3 merge + W^UV + branch sum (+ the TP all-reduce). value = whole-job
ALGORITHMIC HBM bytes per second (sum over ranks of n * per_device_load * d_h * 2 per
sequence, attnkit/costs.py:70-102), so it scales with the work done; ms_per_step is the
step time (max over ranks). Inputs: synthetic bf16 caches with the RMS of the
reference's latents; two distinct cache copies are alternated so every step's working
set is larger than L2 (126 MB) and was not touched by the previous step.

--impl reference: the reference's decode path restated on the host CPU (numpy float64,
oracle/attnkit_port.py, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLRA-4 decode attn µs/step & achieved HBM GB/s per GPU at TP4, 32K ctx vs MLA"
CTX = 32768
BATCH_PER_GROUP = 16


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def peaks_bf16():
    """Measured dense bf16 TFLOP/s (MEASURED_PEAKS.json, burst) or the guide's 2250 nominal."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 2250.0


def ncu_traffic(workload: str):
    """dram read+write bytes per launch of K2 from the committed ncu capture, if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workloads
def make_engine(cfg, own, batch, ctx, seed, device, page_size=128, weights=None, ragged=False):
    """DecodeEngine with a synthetic cache filled on the device (RMS like the reference's rows)."""
    import torch

    from paper_2603_02188_b200 import DecodeEngine
    from paper_2603_02188_b200.costs import calib_factors

    g = torch.Generator(device=device).manual_seed(seed)
    rng = np.random.default_rng(seed)
    if weights is not None:
        w = weights
    elif cfg.variant == "gla" or (cfg.variant == "mlra" and cfg.branches == 2):  # per-group up-projections
        r, dg = cfg.h // cfg.g, cfg.d_c // cfg.g
        w = {f"{n}_{j}": rng.standard_normal((dg, r * cfg.d_h)) * 0.02 for n in ("w_uk", "w_uv") for j in range(cfg.g)}
    else:
        w = {"w_uk": rng.standard_normal((cfg.d_c, cfg.h * cfg.d_h)) * 0.02,
             "w_uv": rng.standard_normal((cfg.d_c, cfg.h * cfg.d_h)) * 0.02}
    eng = DecodeEngine(cfg, w, own, batch=batch, max_tokens=ctx + 64, page_size=page_size, device=device,
                       ragged=ragged)
    lay = eng.layout
    akv = calib_factors(cfg).alpha_kv
    # rope ~ N(0, d * sigma^2) ~ N(0, 1.2) at d = 3072, sigma = 0.02
    pool = eng.cache.pool
    chunk = 1 << 20
    for s in range(0, pool.shape[0], chunk):
        e = min(pool.shape[0], s + chunk)
        blk = torch.randn((e - s, lay.width), generator=g, device=device, dtype=torch.float32)
        blk[:, : lay.nb * lay.dlp] *= akv  # alpha_kv * rmsnorm(.): per-element RMS alpha_kv
        blk[:, lay.nb * lay.dlp:] *= 1.1
        pool[s:e] = blk.to(torch.bfloat16)
    eng.cache.seqlens.fill_(ctx)
    eng.cache._host_lens = [ctx] * batch
    eng.src_weights = w  # the float64 W^UK / W^UV the packs came from (parity tests' oracle input)
    hl = len(eng.heads)
    qn = (torch.randn((batch, hl, cfg.d_h), generator=g, device=device) * 2.0).to(torch.bfloat16)
    qr = torch.zeros((batch, hl, lay.drp), dtype=torch.bfloat16, device=device)
    qr[..., : lay.dr] = torch.randn((batch, hl, lay.dr), generator=g, device=device).to(torch.bfloat16)
    return eng, qn, qr


class StepRunner:
    """Two engines over distinct caches, alternated (A, B, A, B, ...: every step's working set
    is a cache L2 has not just seen). Steps are captured in CUDA graphs: one graph of
    GRAPH_STEPS alternating steps (as a serving loop captures its decode step with the rest
    of the model, amortising the graph launch), plus single-step graphs for remainders."""

    GRAPH_STEPS = 10

    def __init__(self, cfg, own, batch, ctx, device, tp_group=None, full_heads=False, reducer=None):
        import torch

        self.torch = torch
        self.engines = [make_engine(cfg, own, batch, ctx, 1000 + i, device) for i in range(2)]
        self.tp_group = tp_group
        self.reducer = reducer  # collective.PeerAllReduce (K5) or None (NCCL all_reduce)
        self.cfg = cfg
        self.heads = list(self.engines[0][0].heads)
        self.full = torch.zeros((batch, cfg.h, cfg.d_h), dtype=torch.float32, device=device) if tp_group else None
        stream = torch.cuda.Stream(device=device)
        for eng, qn, qr in self.engines:  # warm (attributes, tensor maps), then capture
            eng.decode_attention(qn, qr)
        torch.cuda.synchronize()
        self.fused_tp = reducer is not None and len(self.heads) == cfg.h
        if self.fused_tp:  # once: the K3-fused TP sum against NCCL on the same step
            import torch.distributed as dist

            eng, qn, qr = self.engines[0]
            ref = eng.decode_attention(qn, qr).clone()
            dist.all_reduce(ref, group=tp_group)
            got = eng.decode_attention_tp(qn, qr, reducer, out=self.full).clone()
            torch.cuda.synchronize()
            ok = torch.tensor([float(torch.allclose(got, ref, rtol=1e-5, atol=1e-6))], device=device)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=tp_group)
            self.fused_tp = ok.item() == 1.0
        self.single = []
        for eng, qn, qr in self.engines:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                self._step(eng, qn, qr)
            self.single.append(gr)
        self.multi = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.multi, stream=stream):
            for i in range(self.GRAPH_STEPS):
                self._step(*self.engines[i % 2])
        torch.cuda.synchronize()

    def _step(self, eng, qn, qr):
        if self.fused_tp:
            # every rank holds every head (MLRA-4 by latent block): the TP sum runs inside K3
            return eng.decode_attention_tp(qn, qr, self.reducer, out=self.full)
        out = eng.decode_attention(qn, qr)
        if self.tp_group is not None:
            import torch.distributed as dist

            if len(self.heads) == self.cfg.h:
                self.full.copy_(out)
            else:
                self.full.zero_()
                self.full[:, self.heads] = out
            if self.reducer is not None:
                self.reducer(self.full)
            else:
                dist.all_reduce(self.full, group=self.tp_group)
        return out

    def run(self, steps):
        """Replay exactly `steps` decode steps (alternating caches)."""
        for _ in range(steps // self.GRAPH_STEPS):
            self.multi.replay()
        for i in range(steps % self.GRAPH_STEPS):
            self.single[i % 2].replay()

    def replay(self, i):
        self.single[i % 2].replay()


def make_gqa_engine(cfg, own, batch, ctx, seed, device):
    """GqaDecodeEngine over a synthetic random bf16 cache (K and V heads ~ N(0, 1))."""
    import torch

    from paper_2603_02188_b200.gqa import GqaDecodeEngine

    g = torch.Generator(device=device).manual_seed(seed)
    eng = GqaDecodeEngine(cfg, own, batch=batch, max_tokens=ctx + 64, page_size=128, device=device)
    pool = eng.cache.pool
    for s0 in range(0, pool.shape[0], 1 << 20):
        e = min(pool.shape[0], s0 + (1 << 20))
        pool[s0:e] = torch.randn((e - s0, pool.shape[1]), generator=g, device=device).to(torch.bfloat16)
    eng.cache.seqlens.fill_(ctx)
    eng.cache._host_lens = [ctx] * batch
    q = eng.prepare_queries(torch.randn((batch, cfg.h, cfg.d_h), generator=g, device=device))
    return eng, q


class GqaStepRunner:
    """GQA comparison variant (2.9B: h=24, g=6, d_h=128): two engines over distinct random
    caches, alternated, one CUDA graph each (K2 GQA + split merge)."""

    def __init__(self, cfg, own, batch, ctx, device):
        import torch

        self.engines, self.graphs = [], []
        for i in range(2):
            self.engines.append(make_gqa_engine(cfg, own, batch, ctx, 2000 + i, device))
        stream = torch.cuda.Stream(device=device)
        for eng, q in self.engines:
            eng.decode_attention(q)
        torch.cuda.synchronize()
        for eng, q in self.engines:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                eng.decode_attention(q)
            self.graphs.append(gr)
        torch.cuda.synchronize()

    def run(self, steps):
        for i in range(steps):
            self.graphs[i % 2].replay()


def time_graph_steps(runner, steps, warmup, rank_sync):
    import torch

    runner.run(warmup)
    rank_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    runner.run(steps)
    e1.record()
    torch.cuda.synchronize()
    rank_sync()
    return e0.elapsed_time(e1) / steps  # ms per step


def time_k2_alone(eng_qs, iters):
    """Average device duration of the dominant kernel (K2) alone, CUDA events on its stream."""
    import torch

    from paper_2603_02188_b200 import ops

    stream = torch.cuda.current_stream()
    preps = []
    for eng, qn, qr in eng_qs:
        q_abs, q_rs = ops.absorb_query(qn, qr, eng.w_uk, eng.nb, eng.dlat, eng.scale)
        c = eng.cache
        outs = ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub,
                                   eng.dls, eng.nsplit)
        preps.append((eng, q_abs, q_rs, outs))
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    per = 10
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):  # K2 alone, alternating the two caches
        for i in range(per):
            eng, q_abs, q_rs, outs = preps[i % 2]
            c = eng.cache
            ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub,
                                eng.dls, eng.nsplit, out=outs)
    g.replay()
    torch.cuda.synchronize()
    reps = max(1, iters // per)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * per)


RAGGED_LENS = [int(1024 * 64 ** (i / 15)) for i in range(16)]  # 1K .. 64K, geometric


def ragged_times(device, args):
    """A ragged batch (16 sequences, 1K..64K tokens, geometric) on one TP4 rank: the uniform split
    grid (every sequence nsplit = 9 CTAs) against the device-side plan (mlra_decode_plan: the
    sequences' tiles balanced over one wave of CTAs). Two engines per mode alternate (L2-cold)."""
    import torch

    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.costs import algorithmic_bytes
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = trained_config("mlra4")
    own = shard_ownership(cfg, 4, 0)
    nbytes = algorithmic_bytes(cfg, 4, RAGGED_LENS)
    res = {"lens": RAGGED_LENS, "algorithmic_bytes": nbytes}
    for mode in ("uniform", "plan"):
        engs = []
        for seed in (21, 22):
            eng, qn, qr = make_engine(cfg, own, len(RAGGED_LENS), max(RAGGED_LENS), seed, device,
                                      ragged=(mode == "plan"))
            eng.cache.seqlens.copy_(torch.tensor(RAGGED_LENS, dtype=torch.int32))
            eng.cache._host_lens = list(RAGGED_LENS)
            engs.append((eng, qn, qr))
        for eng, qn, qr in engs:
            eng.decode_attention(qn, qr)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            for i in range(10):
                eng, qn, qr = engs[i % 2]
                eng.decode_attention(qn, qr)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        res[mode] = {"us_per_step": round(us, 2), "gbs": round(nbytes / (us * 1e-6) / 1e9, 1),
                     "nsplit": engs[0][0].nsplit}
        del engs, g
        torch.cuda.empty_cache()
    res["speedup"] = round(res["uniform"]["us_per_step"] / res["plan"]["us_per_step"], 3)
    return res


def time_paper_scope(eng_qs, iters=40):
    """The paper's decode-attention scope (Eq. step-2 decoding): absorbed queries in,
    latent mixture Z out -- K2 + the split merge (K3 with upproj = 0), no absorption (Step 1) and no
    W^UV up-projection (Step 3). One CUDA graph of 10 steps alternating the two caches."""
    import torch

    from paper_2603_02188_b200 import ops

    preps = []
    for eng, qn, qr in eng_qs:
        q_abs, q_rs = ops.absorb_query(qn, qr, eng.w_uk, eng.nb, eng.dlat, eng.scale)
        c = eng.cache
        parts = ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub,
                                    eng.dls, eng.nsplit)
        z = ops.combine(*parts, None, 1.0)
        preps.append((eng, q_abs, q_rs, parts, z))
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for i in range(10):
            eng, q_abs, q_rs, parts, z = preps[i % 2]
            c = eng.cache
            ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub,
                                eng.dls, eng.nsplit, out=parts)
            ops.combine(*parts, None, 1.0, out=z)
    g.replay()
    torch.cuda.synchronize()
    reps = max(1, iters // 10)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * 10)


def e2e_steps(engines, steps, warmup, reducer=None, rank_sync=None):
    """The plugin calls a user makes, with HOST buffers, every step: one H2D of the new token's
    cache rows + queries from pinned memory, K0 (append, advancing seqlens) + K1..K3 through
    the C ABI (with reducer: mlra_decode_step_tp, the TP group's sum fused into K3), one D2H of
    the fp32 output. Two micro-batches (the two caches) are stepped in turn by
    host_loop.MicroBatchLoop: micro-batch k+1's upload and k-1's download overlap k's kernels.
    Also returns the serial time (one micro-batch, copies in line on one stream). Under torchrun
    every rank runs it (same call sequence); the caller takes the max over ranks."""
    import torch

    from paper_2603_02188_b200 import ops
    from paper_2603_02188_b200.host_loop import MicroBatchLoop

    sync = rank_sync or torch.cuda.synchronize
    loop = MicroBatchLoop(engines, reducer=reducer, graphs=True)
    g = torch.Generator().manual_seed(7)
    for k in range(len(loop)):
        for t in loop.host_inputs(k):
            t.copy_(torch.randn(t.shape, generator=g).to(torch.bfloat16))
    start_lens = [e.cache.lengths() for e in engines]

    def run(n):
        for i in range(n):
            loop.submit(i % len(loop))

    run(warmup * len(loop))
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    loop.start()
    t0 = time.perf_counter()
    e0.record()
    run(steps)
    loop.join()
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    sync()
    piped = max(e0.elapsed_time(e1) / 1e3, wall) / steps

    # serial reference point: same calls, one micro-batch, every copy in line
    eng = engines[0]
    c = eng.cache
    h_in = loop.host_inputs(0)
    d_in = [torch.empty_like(t, device=eng.device) for t in h_in]
    h_out = loop.host_output(0)

    def one():
        for d, h in zip(d_in, h_in):
            d.copy_(h, non_blocking=True)
        c.reserve_token()
        ops.cache_append(d_in[0], c.block_table, c.seqlens, c.pool, c.page_size, advance=True)
        out = eng.decode_attention_tp(d_in[1], d_in[2], reducer) if reducer is not None else \
            eng.decode_attention(d_in[1], d_in[2])
        h_out.copy_(out, non_blocking=True)

    nser = max(3, steps // 2)
    for _ in range(warmup):
        one()
    sync()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(nser):
        one()
    e1.record()
    torch.cuda.synchronize()
    serial = max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0) / nser
    sync()
    for e, lens in zip(engines, start_lens):  # back to the benchmark context
        e.cache.seqlens.copy_(torch.tensor(lens, dtype=torch.int32))
        e.cache._host_lens = list(lens)
    bin_, bout = loop.bytes_per_step(0)
    return piped, serial, bin_, bout


# ----------------------------------------------------------------------------- CPU side
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_sample(phi: int, n: int, seqs: int, seed: int = 0):
    """Time the oracle port's attention (attend_local + reduce) over `seqs` sequences of n tokens
    (the fallback CPU baseline when the reference is not installed in baseline/_ref)."""
    from oracle import attnkit_port as ak

    cfg = ak.Cfg("mlra", 24, 3072, 128, 64, 512, 1024, branches=4, scaling=True)
    rng = np.random.default_rng(seed)
    w = {"w_uk": rng.standard_normal((512, 24 * 128)) * 0.02, "w_uv": rng.standard_normal((512, 24 * 128)) * 0.02}
    units = ak.shard_units(cfg, phi, 0)[1]
    streams = {"rope": rng.standard_normal((n, 64))}
    for _, _g, b, _h in units:
        streams[f"latent_b{b}"] = rng.standard_normal((n, 128)) * 24 ** 0.5 / 8
    qn = rng.standard_normal((24, 128))
    qr = rng.standard_normal((24, 64))
    t0 = time.perf_counter()
    for _ in range(seqs):
        ak.reduce_contributions(cfg, ak.attend_latent(cfg, w, ak.Cache(dict(streams)), qn, qr, units))
    dt = time.perf_counter() - t0
    per_tok_bytes = (len(units) * 128 + 64) * 2
    return seqs * n * per_tok_bytes / dt / 1e9, dt


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The unmodified reference package (attnkit), installed into baseline/_ref by
    `pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of
    /root/reference/pkg>`; None when absent."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import attnkit
        from attnkit import cache as ak_cache
        from attnkit import decode as ak_decode
        from attnkit import tpsim as ak_tpsim
    except Exception:
        return None
    return attnkit, ak_cache, ak_decode, ak_tpsim


class ReferenceWorkload:
    """The reference's own decode attention (attnkit/decode.py:204-285) over a batch of
    sequences of one TP group: per sequence and per logical device of the group, attnkit's
    ``attend_local`` on that device's ``KvCache`` (built once with ``cache_from_streams``,
    attnkit/cache.py:95-102; random rows with the RMS of the reference's latents), then one
    ``reduce_contributions`` over the devices' contributions in device-id order -- the body of
    ``sim_decode`` (attnkit/tpsim.py:269-276) without the token append. Sequences run one after
    the other on the reference's stock path (its ATTNKIT_THREADS default is 1 worker; numpy's
    BLAS uses every host thread)."""

    def __init__(self, ref, phi: int, seqs: int, n: int, seed: int = 0):
        attnkit, ak_cache, ak_decode, ak_tpsim = ref
        self.ak_decode = ak_decode
        self.cfg = attnkit.trained_config("mlra4")
        cfg = self.cfg
        rng = np.random.default_rng(seed)
        w = {"w_uk": rng.standard_normal((cfg.d_c, cfg.h * cfg.d_h)) * 0.02,
             "w_uv": rng.standard_normal((cfg.d_c, cfg.h * cfg.d_h)) * 0.02}
        self.devices = []
        for k in range(phi):
            own = ak_tpsim.shard_ownership(cfg, phi, k) if phi > 1 else ak_decode.full_ownership(cfg)
            self.devices.append((own, ak_decode.local_weights(cfg, w, own)))
        akv = (4 * cfg.d / cfg.d_c) ** 0.5  # alpha_kv: the cached latent's per-element RMS
        self.caches = []
        for _ in range(seqs):
            rope = rng.standard_normal((n, cfg.d_h_rope)) * 1.1
            per_dev = []
            for own, _lw in self.devices:
                streams = {u.stream: rng.standard_normal((n, cfg.block_dim)) * akv for u in own.units}
                streams["rope"] = rope
                per_dev.append(ak_cache.cache_from_streams(cfg, streams))
            self.caches.append(per_dev)
        self.queries = {"q_nope": rng.standard_normal((cfg.h, cfg.d_h)),
                        "q_rope": rng.standard_normal((cfg.h, cfg.d_h_rope))}
        self.bytes_per_step = seqs * n * sum((len(own.units) * cfg.block_dim + cfg.d_h_rope) * 2
                                             for own, _ in self.devices)

    def step(self):
        d = self.ak_decode
        for per_dev in self.caches:
            contribs = []
            for (own, lw), cache in zip(self.devices, per_dev):
                contribs.extend(d.attend_local(self.cfg, lw, own, cache, self.queries))
            d.reduce_contributions(self.cfg, contribs)


def cpu_baseline():
    """The reference's own CPU path (attnkit, baseline/_ref) on a bounded sample of the N = 1
    workload: 6 sequences x 32K (TP1), attended twice (~5-10 s of host work); the oracle port
    when the reference is not installed."""
    ref = import_reference()
    if ref is None:
        nseq = BATCH_PER_GROUP * 16
        gbs_cpu, dt = cpu_oracle_sample(1, CTX, nseq)
        return {"value": round(gbs_cpu, 3), "unit": "GB/s", "cores": cpu_cores(), "kind": "port",
                "sample": f"{nseq} sequences x {CTX} tokens of the TP1 workload (numpy float64 oracle "
                          f"attend_local+reduce, BLAS on all host threads), {dt:.1f} s"}
    work = ReferenceWorkload(ref, 1, 6, CTX, seed=1)
    work.step()
    t0 = time.perf_counter()
    for _ in range(2):
        work.step()
    dt = time.perf_counter() - t0
    return {"value": round(2 * work.bytes_per_step / dt / 1e9, 4), "unit": "GB/s", "cores": cpu_cores(),
            "kind": "reference", "sample": f"2 x 6 sequences x {CTX} tokens of the TP1 workload: attnkit "
                                           f"attend_local + reduce_contributions (baseline/_ref, float64, BLAS on "
                                           f"all host threads), {dt:.1f} s"}


# ----------------------------------------------------------------------------- main
def run_reference(args):
    """--impl reference: the reference's own CPU path (attnkit from baseline/_ref, unmodified)
    on this arm's workload, rank 0 only. N = 1: the whole configs[1] batch (16 sequences x 32K,
    TP1) every step. N > 1: each step a bounded sample of the TP-group workload (4 sequences x
    32K on all phi logical devices; the full group would take minutes per step on the host)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = import_reference()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n_gpus = world if world > 1 else args.gpus
    phi = 1 if n_gpus == 1 else min(n_gpus, 4)
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "attnkit not installed in baseline/_ref"}))
        return 0
    seqs = BATCH_PER_GROUP if n_gpus == 1 else 4
    ctx = context_for(n_gpus)
    t_build = time.perf_counter()
    work = ReferenceWorkload(ref, phi, seqs, ctx)
    t_build = time.perf_counter() - t_build
    for _ in range(args.warmup):
        work.step()
    times = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ts = time.perf_counter()
        work.step()
        times.append(time.perf_counter() - ts)
    total = time.perf_counter() - t0
    ms = total / args.steps * 1e3
    gbs = work.bytes_per_step / (ms * 1e-3) / 1e9
    sample = (f"{seqs} sequences x {ctx} tokens per step on {phi} logical device(s): attnkit attend_local per "
              f"(sequence, device) + reduce_contributions (float64 numpy, BLAS on all host threads); "
              f"{'the whole batch' if n_gpus == 1 else 'a bounded sample of the group batch'}; caches built "
              f"once with cache_from_streams ({t_build:.1f} s, untimed)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong" if n_gpus <= 4 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random rows with the reference latents' RMS)",
        "config": {"workload": _workload_name(n_gpus), "model": "2.9B MLRA-4 attention layer (h=24, d_h=128, "
                   "d_c=512, d_h^R=64)", "global_batch": seqs, "seq_len": ctx,
                   "parallelism": f"tp{phi} (simulated devices, attnkit/tpsim.py)" if phi > 1 else "tp1",
                   "reference": "attnkit 0.1.0, unmodified (baseline/_ref)"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cpu_cores(), "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_ms_min_median": [round(min(times) * 1e3, 3), round(float(np.median(times)) * 1e3, 3)],
        "wall_s": round(total, 2),
    }
    print(json.dumps(line))
    return 0


def context_for(n_gpus: int) -> int:
    """configs[2] (TP4 on 4 GPUs) is quoted at 64K; every other N runs the 32K metric context."""
    return 65536 if n_gpus == 4 else CTX


def _workload_name(n):
    return {1: "configs[1]: MLRA-4 2.9B layer, B=16, 32K ctx, TP1 on 1 GPU",
            2: "MLRA-4 2.9B layer, B=16, 32K ctx, TP2 (rank sum fused into K3 over NVLink peer memory)",
            4: "configs[2]: MLRA-4 2.9B layer, B=16, 64K ctx, TP4 (rank sum fused into K3 over NVLink peer "
               "memory; NCCL all-reduce only as the fallback)",
            8: "configs[4]: 2 x TP4 over B=32 (16 per group), 32K ctx (rank sum fused into K3)"}.get(n, f"{n} GPUs")


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.costs import algorithmic_bytes
    from paper_2603_02188_b200.tp import group_ranks, shard_ownership

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = world if world > 1 else args.gpus
    # test hook: MLRA_BENCH_SHARED_GPU=1 runs every rank on cuda:0 over gloo (the multi-rank
    # path exercised on a one-GPU box; time-sliced contexts, not a performance measurement)
    shared = os.environ.get("MLRA_BENCH_SHARED_GPU") == "1"
    dev_index = 0 if shared else local_rank
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    tp = 1 if n_gpus == 1 else min(n_gpus, 4)
    groups = None
    if world > 1:
        groups = [dist.new_group(r) for r in group_ranks(world, tp)]

    def rank_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    cfg = trained_config("mlra4")
    own = shard_ownership(cfg, tp, rank % tp)
    tp_group = groups[rank // tp] if groups else None
    reducer, allreduce_kind = None, "none (tp1)"
    if tp_group is not None:
        reducer, allreduce_kind = make_reducer(args.allreduce, tp_group, BATCH_PER_GROUP * cfg.h * cfg.d_h, device)
    ctx = context_for(n_gpus)
    runner = StepRunner(cfg, own, BATCH_PER_GROUP, ctx, device, tp_group=tp_group, reducer=reducer)
    with ClockSampler(dev_index) as clk:
        ms = time_graph_steps(runner, args.steps, args.warmup, rank_sync)
        # K2's launch duration for the roofline, timed alone right after the timed steps (same
        # engines, same clocks; not after the e2e run below, whose load sits at the power cap)
        k2_ms = time_k2_alone(runner.engines, 40) if rank == 0 else 0.0
        t = torch.tensor([ms], device=device)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # The timed region can be only milliseconds long: keep replaying the same step
        # (untimed, same count on every rank) for ~0.6 s so the clock record sees real load.
        runner.run(max(50, int(600.0 / max(ms, 1e-3))))
        rank_sync()
    bytes_rank = algorithmic_bytes(cfg, tp, [ctx] * BATCH_PER_GROUP)
    total_bytes = bytes_rank * n_gpus
    value = total_bytes / (ms * 1e-3) / 1e9

    # end to end through the C ABI from pinned host buffers, on every rank (the TP sum fused
    # into K3 when the group has one); whole-job bytes over the slowest rank's time
    e2e_red = reducer if runner.fused_tp else None
    # (at least 40 steps: the steady-state rate of a serving loop, the pipeline fill amortised)
    e2e_s, ser_s, bin_, bout = e2e_steps([e for e, _, _ in runner.engines], max(40, args.steps), args.warmup,
                                         reducer=e2e_red, rank_sync=rank_sync)
    tt = torch.tensor([e2e_s, ser_s], device=device)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s, ser_s = float(tt[0]), float(tt[1])

    extras = {}
    if rank == 0:
        hbm_peak, peak_kind = peaks()
        k2_bytes = bytes_rank
        achieved = k2_bytes / (k2_ms * 1e-3) / 1e9
        workload = f"mlra4_tp{tp}_b{BATCH_PER_GROUP}_n{ctx}"
        extras["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                              "frac": round(achieved / hbm_peak, 4), "traffic": ncu_traffic(workload),
                              "kernel": "mlra_decode_kernel (K2)", "kernel_us": round(k2_ms * 1e3, 2),
                              "algorithmic_bytes_per_launch": k2_bytes, "peak_kind": f"{peak_kind} copy (burst)"}
        extras["clocks"] = clk.summary()
        if n_gpus == 1 and not args.quick:
            extras.update(per_gpu_comparisons(cfg, device, args))
        if n_gpus == 1 and not args.no_cpu:
            extras["cpu_baseline"] = cpu_baseline()
        extras["e2e"] = {"value": round(total_bytes / e2e_s / 1e9, 1), "unit": "GB/s", "h2d_bytes_per_step": bin_,
                         "d2h_bytes_per_step": bout, "ms_per_step": round(e2e_s * 1e3, 4),
                         "serial_ms_per_step": round(ser_s * 1e3, 4),
                         "path": "host_loop.MicroBatchLoop: per step 1 H2D (pinned rows+queries), mlra_cache_append "
                                 "(advance) + " + ("mlra_decode_step_tp (C ABI; the TP sum over the group fused into K3)"
                                                   if e2e_red is not None else "mlra_decode_step (C ABI)") +
                                 " (captured once per micro-batch after its first step and replayed from a CUDA "
                                 "graph), 1 D2H; 2 micro-batches, the copies and K0 on side streams overlapping the other "
                                 "micro-batch's kernels; serial_ms_per_step = same calls on one stream, no overlap; "
                                 "per-rank bytes/step and Bi/Bo, time = max over ranks"}
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "strong" if n_gpus <= 4 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random bf16 caches with the reference's latent RMS; random W^UK/W^UV)",
            "config": {"workload": _workload_name(n_gpus), "model": "2.9B MLRA-4 attention layer (h=24, d_h=128, "
                       "d_c=512, d_h^R=64)", "global_batch": BATCH_PER_GROUP * max(1, n_gpus // 4), "seq_len": ctx,
                       "parallelism": f"tp{tp}" + (f"xdp{n_gpus // tp}" if n_gpus > tp else ""),
                       "l2": "2 distinct caches alternated; per-step working set > 126 MB L2",
                       "graphs": "10 alternating steps per CUDA graph replay",
                       "allreduce": allreduce_kind + ("; fused into K3 (checked against NCCL)" if runner.fused_tp
                                                      else ""),
                       "algorithmic_bytes_per_gpu_per_step": bytes_rank, "page_size": 128,
                       "nsplit": runner.engines[0][0].nsplit},
            "gpu_launches": (3 + (1 if reducer is not None and not runner.fused_tp else 0)) * args.steps,
        }
        line.update(extras)
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def median_ms(runner, args, reps=3):
    """Comparison rows: median of three timed loops (the SM clock moves under the power cap)."""
    import statistics

    import torch

    return statistics.median(time_graph_steps(runner, args.steps, args.warmup, torch.cuda.synchronize)
                             for _ in range(reps))


def per_gpu_comparisons(cfg, device, args):
    """The headline per-GPU numbers on one device: one TP4 rank of MLRA-4 (block + rope) and
    the MLA baseline at the same shapes (TP4 heads-sharded rank: full latent, 6 heads; and TP1)."""
    import torch

    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.costs import algorithmic_bytes
    from paper_2603_02188_b200.tp import shard_ownership

    out = {}
    mla = trained_config("mla")
    cases = {
        "mlra4_tp4_rank": (cfg, shard_ownership(cfg, 4, 0), 4),
        "mla_tp4_rank": (mla, shard_ownership(mla, 4, 0), 4),
        "mla_tp1": (mla, None, 1),
    }
    res = {}
    for name, (c, own, phi) in cases.items():
        r = StepRunner(c, own, BATCH_PER_GROUP, CTX, device)
        ms = median_ms(r, args)
        nbytes = algorithmic_bytes(c, phi, [CTX] * BATCH_PER_GROUP)
        ps = time_paper_scope(r.engines)
        res[name] = {"us_per_step": round(ms * 1e3, 2), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                     "algorithmic_bytes": nbytes, "paper_scope_us": round(ps * 1e3, 2),
                     "paper_scope_gbs": round(nbytes / (ps * 1e-3) / 1e9, 1)}
        del r
        torch.cuda.empty_cache()
    out["tp4_per_gpu"] = res["mlra4_tp4_rank"]
    out["vs_mla"] = {
        "mla_tp4_rank_us": res["mla_tp4_rank"]["us_per_step"],
        "mlra4_tp4_rank_us": res["mlra4_tp4_rank"]["us_per_step"],
        "speedup_per_gpu_tp4": round(res["mla_tp4_rank"]["us_per_step"] / res["mlra4_tp4_rank"]["us_per_step"], 3),
        "mla_tp1_us": res["mla_tp1"]["us_per_step"], "mla_tp1_gbs": res["mla_tp1"]["gbs"],
        "paper_claim": "~2.8x (H100, FlashMLA vs FA3-based MLRA-4)", "traffic_ratio": 3.0,
        "paper_scope": {
            "what": "the paper's decode-attention scope (PAPER.md:551, Eq. step-2): absorbed queries in, latent "
                    "mixture out = K2 + split merge, without the W^UK absorption (Step 1) and the W^UV "
                    "up-projection (Step 3)",
            "mlra4_tp4_rank_us": res["mlra4_tp4_rank"]["paper_scope_us"],
            "mla_tp4_rank_us": res["mla_tp4_rank"]["paper_scope_us"],
            "speedup_per_gpu_tp4": round(res["mla_tp4_rank"]["paper_scope_us"] /
                                         res["mlra4_tp4_rank"]["paper_scope_us"], 3)},
    }
    # GQA baseline (2.9B, g=6: K and V heads, 3072 B/token at TP1, 1536 B/token per TP2 rank)
    gqa = trained_config("gqa")
    g_res = {}
    for name, own, phi in (("gqa_tp1", None, 1), ("gqa_tp2_rank", shard_ownership(gqa, 2, 0), 2)):
        r = GqaStepRunner(gqa, own, BATCH_PER_GROUP, CTX, device)
        ms = median_ms(r, args)
        nbytes = algorithmic_bytes(gqa, phi, [CTX] * BATCH_PER_GROUP)
        g_res[name] = {"us_per_step": round(ms * 1e3, 2), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                       "algorithmic_bytes": nbytes}
        del r
        torch.cuda.empty_cache()
    # the other latent variants on the same kernels, per TP rank
    v_res = {}
    for name, phi in (("mlra2", 4), ("gla2", 2)):
        c = trained_config(name)
        r = StepRunner(c, shard_ownership(c, phi, 0), BATCH_PER_GROUP, CTX, device)
        ms = median_ms(r, args)
        nbytes = algorithmic_bytes(c, phi, [CTX] * BATCH_PER_GROUP)
        v_res[f"{name}_tp{phi}_rank"] = {"us_per_step": round(ms * 1e3, 2), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                                         "algorithmic_bytes": nbytes}
        del r
        torch.cuda.empty_cache()
    out["latent_variants"] = v_res
    out["vs_gqa"] = {
        "gqa_tp1": g_res["gqa_tp1"], "gqa_tp2_rank": g_res["gqa_tp2_rank"],
        "mlra4_tp4_rank_us": res["mlra4_tp4_rank"]["us_per_step"],
        "speedup_per_gpu_mlra4_tp4_vs_gqa_tp2": round(g_res["gqa_tp2_rank"]["us_per_step"] /
                                                      res["mlra4_tp4_rank"]["us_per_step"], 3),
        "traffic_ratio_gqa_tp2_rank_vs_mlra4_tp4_rank": 4.0,
    }
    out["layer"] = layer_times(device, args)
    out["ragged"] = ragged_times(device, args)
    out["output_side"] = output_side_times(device)
    out["prefill"] = prefill_times(device)
    return out


def make_layer_engine(cfg, own, batch, ctx, seed, device, page_size=128):
    """DecodeEngine with the FULL weight set of the layer (weights.py shapes, sigma 0.02: the
    projections as well as W^UK / W^UV) and a synthetic cache of ctx tokens, plus the new
    tokens' hidden rows [B, d] ~ N(0, 1) for decode_layer."""
    import torch

    from paper_2603_02188_b200.weights import weight_shapes

    rng = np.random.default_rng(seed)
    w = {name: rng.standard_normal(shape) * 0.02 for name, shape in weight_shapes(cfg).items()}
    eng, _, _ = make_engine(cfg, own, batch, ctx, seed, device, page_size=page_size, weights=w)
    g = torch.Generator(device=device).manual_seed(seed + 1)
    hidden = torch.randn((batch, cfg.d), generator=g, device=device)
    return eng, hidden


def layer_times(device, args):
    """The attention layer from the hidden rows (the paper's end-to-end decode scope: pre-attention
    plus attention), B = 16, 32K, per GPU: K-1 down -> K0 -> K-1 query -> [K1] ->
    K2 -> K3 (hand-written K-1; the TP4 rank's query kernel writes q~ with W^UQ.W^UK_b
    pre-multiplied, so K1 is skipped), against the same step with the projections as torch
    bf16 cuBLAS GEMMs + rmsnorm / rope ops (K0-K3 unchanged). Two engines alternate (L2-cold
    caches and weights); the timing loop rewrites the appended slot (advance=False), so the
    attended length stays ctx."""
    import torch

    from paper_2603_02188_b200 import ops
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.projections import rope_rotate
    from paper_2603_02188_b200.tp import shard_ownership

    def gtime(fns, reps=20):
        for f in fns:
            f()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(10):
                fns[i % len(fns)]()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 10 * 1e3

    cfg = trained_config("mlra4")
    res = {}
    for name, own in (("mlra4_tp4_rank", shard_ownership(cfg, 4, 0)), ("mlra4_tp1", None)):
        engs = [make_layer_engine(cfg, own, BATCH_PER_GROUP, CTX, 11 + i, device) for i in range(2)]
        for eng, _ in engs:
            eng.kernel_projector(None)
        kp = engs[0][0].kernel_projector(None)

        def layer(i):
            eng, hid = engs[i]
            return lambda: eng.decode_layer(hid, advance=False)

        def proj(i):
            eng, hid = engs[i]
            k = eng.kernel_projector(None)

            def f():
                k.down(hid)
                k.query(hid.shape[0], eng.cache.seqlens)
            return f

        def attn(i):
            eng, hid = engs[i]
            qn = torch.randn((BATCH_PER_GROUP, len(eng.heads), cfg.d_h), device=device).to(torch.bfloat16)
            qr = torch.zeros((BATCH_PER_GROUP, len(eng.heads), eng.layout.drp), dtype=torch.bfloat16, device=device)
            return lambda: eng.decode_attention(qn, qr)

        def torch_layer(i):
            eng, hid = engs[i]
            k = eng.kernel_projector(False)  # q_nope weights (W^UQ) for the cuBLAS query GEMM
            c = eng.cache
            from paper_2603_02188_b200.decode import _write_plan
            _, blocks, block0, nblocks, ng = _write_plan(cfg, eng.own)
            pos = c.seqlens.long()

            def f():
                y = torch.mm(hid.to(torch.bfloat16), k.w_down, out_dtype=torch.float32)
                cq = y[:, :k.n_q]
                kv, kr = y[:, k.n_q:k.n_q + k.n_kv].contiguous(), y[:, k.n_q + k.n_kv:k.n_q + k.n_kv + k.n_kr].contiguous()
                ops.cache_append_latent(kv, kr, None, c.seqlens, c.block_table, c.pool, c.page_size, branches=blocks,
                                        block0=block0, nblocks=nblocks, dlp=eng.layout.dlp, drp=eng.layout.drp,
                                        alpha_kv=k.alpha_kv, norm_groups=ng, advance=False)
                cq = k.alpha_q * cq * torch.rsqrt((cq * cq).mean(-1, keepdim=True) + 1e-6)
                q = torch.mm(cq.to(torch.bfloat16), k.w_query, out_dtype=torch.float32)
                qn = q[:, :k.nq].reshape(-1, k.H, cfg.d_h).to(torch.bfloat16)
                qr = torch.zeros((qn.shape[0], k.H, eng.layout.drp), dtype=torch.bfloat16, device=device)
                qr[..., :k.dr] = rope_rotate(q[:, k.nq:k.nq + k.H * k.dr].reshape(-1, k.H, k.dr), pos).to(torch.bfloat16)
                eng.decode_attention(qn, qr)
            return f

        t_layer = gtime([layer(0), layer(1)])
        t_proj = gtime([proj(0), proj(1)])
        t_attn = gtime([attn(0), attn(1)])
        t_torch = gtime([torch_layer(0), torch_layer(1)])
        wbytes = (kp.w_down.numel() + kp.w_query.numel()) * 2  # algorithmic: the unpadded weights
        res[name] = {"layer_us": round(t_layer, 2), "k_minus1_us": round(t_proj, 2),
                     "k_minus1_weight_bytes": wbytes, "k_minus1_gbs": round(wbytes / (t_proj * 1e-6) / 1e9, 1),
                     "attention_step_us": round(t_attn, 2), "layer_torch_projections_us": round(t_torch, 2),
                     "query_preabsorbed": bool(kp.absorbed)}
        del engs
        torch.cuda.empty_cache()
    return res


def prefill_times(device):
    """latent_prefill's device part for one 2.9B MLRA-4 sequence at TP1 (random weights): the n-row
    projections (cuBLAS bf16 + fused split / rope epilogues), K0 over all tokens, the batched
    absorption GEMM and K6 (tcgen05 causal prefill); K6 alone against the measured bf16 tensor peak
    (algorithmic FLOPs: 2*(d_lat + d_rope + d_lat) per causal (query, key) pair per head and branch,
    plus the in-kernel W^UV up-projection); and the previous n-pseudo-sequence decode path at 4096."""
    import torch

    from paper_2603_02188_b200 import decode as dec
    from paper_2603_02188_b200 import ops
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.weights import weight_shapes

    cfg = trained_config("mlra4")
    rng = np.random.default_rng(0)
    w = {name: rng.standard_normal(shape) * 0.02 for name, shape in weight_shapes(cfg).items()}
    st = dec._state(cfg, w, device)
    tflops_peak = peaks_bf16()

    def ev(fn, reps=3):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts[1:])

    res = {}
    for n in (1024, 4096, 16384):
        h_t = torch.randn((n, cfg.d), device=device)
        cache = dec.new_cache(cfg, device=device, initial_tokens=n)
        ms = ev(lambda: dec.prefill_into(cfg, st, cache, h_t))
        kp = st.kproj
        _, _, qn, q_r = kp.project_gemm(h_t, 0, drq=64)
        w_uk, w_uv = st.lw.packed(cache.layout, device, st.own)
        q_abs = torch.bmm(qn.transpose(0, 1), w_uk).view(cfg.h, n, 4, 128)
        q_rs = (q_r.float() * ops.score_scale(cfg.tau)).to(torch.bfloat16)
        pc = cache.paged
        k6 = ev(lambda: ops.prefill_attention(q_abs, q_rs, w_uv, pc.pool, pc.block_table, pc.page_size, 4, 128, 64,
                                              0.5))
        flops = 4 * cfg.h * (n * (n + 1) / 2) * 2 * (128 + 64 + 128) + n * cfg.h * 4 * 128 * 128 * 2 * 2
        row = {"ms": round(ms, 3), "tokens_per_s": round(n / (ms * 1e-3), 1), "k6_ms": round(k6, 3),
               "k6_tflops": round(flops / (k6 * 1e-3) / 1e12, 1),
               "k6_frac_of_bf16_peak": round(flops / (k6 * 1e-3) / 1e12 / tflops_peak, 3)}
        if n == 4096:
            row["pseudo_sequence_path_ms"] = round(ev(lambda: dec.prefill_into(cfg, st, cache, h_t,
                                                                               force_pseudo=True), reps=2), 3)
        res[f"n{n}"] = row
        del cache
        torch.cuda.empty_cache()
    res["roofline"] = {"bound": "tensor", "peak_tflops": tflops_peak, "peak_kind": "measured cuBLAS bf16 (burst)"}
    return res


def output_side_times(device):
    """K4a + K4 (gate, W_o, residual; world 1) against the torch path (sigmoid, cast, cuBLAS
    GEMM, add) at the step's batch: an MLRA-4 TP4 rank holds a partial of all 24 heads (K =
    3072), an MLA TP4 rank 6 heads (K = 768); d = 3072. Eight W_o copies are cycled so W_o
    comes from HBM (8 x 18.9 MB > L2). The multi-rank all-reduce needs peers (not timed here)."""
    import torch

    from paper_2603_02188_b200 import ops

    def gtime(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 10 * 1e3

    res = {}
    B, D = BATCH_PER_GROUP, 3072
    for name, K in (("mlra4_tp4_rank", 3072), ("mla_tp4_rank", 768)):
        attn, gate = torch.randn(B, K, device=device), torch.randn(B, K, device=device)
        w_os = [torch.randn(K, D, device=device).to(torch.bfloat16) for _ in range(8)]
        resid, y = torch.randn(B, D, device=device), torch.empty(B, D, device=device)
        ws = ops.outproj_workspace(B, K, device)
        it = [0]

        def k4():
            it[0] += 1
            ops.outproj(attn, gate, w_os[it[0] % 8], resid, y, workspace=ws)

        def ref():
            it[0] += 1
            y.copy_(resid + ((attn * torch.sigmoid(gate)).to(torch.bfloat16) @ w_os[it[0] % 8]).float())

        t4, tr = gtime(k4), gtime(ref)
        res[name] = {"K": K, "k4_us": round(t4, 2), "torch_us": round(tr, 2),
                     "w_o_gbs": round(K * D * 2 / (t4 * 1e-6) / 1e9, 1)}
        del w_os
        torch.cuda.empty_cache()
    return res


def make_reducer(kind, group, n, device):
    """The TP step's sum over ranks: K5 over NVLink peer memory (default) or NCCL. K5 is checked
    once against NCCL on a random buffer; any failure or mismatch falls back to NCCL (recorded)."""
    import torch
    import torch.distributed as dist

    if kind == "nccl":
        return None, "nccl all_reduce"
    try:
        from paper_2603_02188_b200.collective import PeerAllReduce

        red = PeerAllReduce(group, n, device)
        g = torch.Generator(device=device).manual_seed(dist.get_rank())
        x = torch.randn(n, generator=g, device=device)
        a, b = x.clone(), x.clone()
        red(a)
        dist.all_reduce(b, group=group)
        torch.cuda.synchronize()
        ok = torch.tensor([float(torch.allclose(a, b, rtol=1e-5, atol=1e-5))], device=device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() == 1.0:
            return red, ("peer (one-shot over NVLink IPC mappings, rank-order sum: fused into K3 via "
                         "mlra_decode_step_tp when every rank holds every head, else K5 mlra_allreduce)")
        red.close()
        return None, "nccl all_reduce (K5 self-check mismatch)"
    except Exception as e:  # IPC / peer access unavailable
        return None, f"nccl all_reduce (K5 unavailable: {type(e).__name__})"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--quick", action="store_true", help="skip the per-GPU TP4 / MLA comparison runs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-oracle baseline sample")
    ap.add_argument("--allreduce", choices=("peer", "nccl"), default="peer",
                    help="TP step sum: K5 over NVLink peer memory (default) or NCCL")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
