"""Parity pinned at EXACTLY the configurations bench.py times.

Every engine here is built by bench.py's own ``make_engine`` / ``make_gqa_engine`` (same
synthetic cache generator, page size 128, default split count: nsplit = 9 at B = 16, 148 at
B = 1), run through the same ``decode_attention`` call the bench captures in its CUDA graphs,
and compared with the float64 oracle evaluated on the SAME bf16 inputs: the cache rows read
back from the pool through the block table, the bf16 weight packs' source rounded to bf16,
and the bf16 queries. Gate: max_rel_err <= 1e-2; the measured errors are
logged (``MLRA_PARITY_LOG=<file>`` appends one JSON line per case) and tabled in DESIGN.md.

Configs: BASELINE configs[1] (TP1, B = 16, 32K), the headline TP4 rank (B = 16, 32K), configs[2]
(TP4 rank, 64K), the MLA and GQA comparison rows, MLRA-2 / GLA-2 rank rows, and long-context
B = 1 points (148 splits).
"""

import json
import os
import sys

import numpy as np
import pytest
import torch

from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-2


def _bench():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import bench

    return bench


def _log(case, errs, extra=None):
    path = os.environ.get("MLRA_PARITY_LOG")
    rec = {"case": case, "max_rel_err_max": float(max(errs)), "max_rel_err_median": float(np.median(errs)),
           "n_seqs": len(errs)}
    if extra:
        rec.update(extra)
    print(json.dumps(rec))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _bf16_weights(w):
    return {k: ak.bf16_round(v) for k, v in w.items()}


def _streams(eng, s):
    """Sequence s's streams as stored in the pool (bf16 values, float64 arrays)."""
    return {name: eng.cache.stream(s, name).double().cpu().numpy() for name in list(eng.layout.units) + ["rope"]}


def _check_latent(variant, phi, rank, batch, ctx, seqs=None, graph=True, cfg=None):
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.tp import shard_ownership

    bench = _bench()
    cfg = cfg if cfg is not None else trained_config(variant)
    own = shard_ownership(cfg, phi, rank) if phi > 1 else None
    dev = torch.device("cuda", 0)
    eng, qn, qr = bench.make_engine(cfg, own, batch, ctx, 1000, dev)
    out = eng.decode_attention(qn, qr).clone()
    if graph:  # the bench replays the step from a CUDA graph: bit-identical to the eager call
        g = torch.cuda.CUDAGraph()
        res = torch.empty_like(out)
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            eng.decode_attention(qn, qr, out=res)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, res)
    got = out.double().cpu().numpy()
    ocfg = ak.cfg_from(cfg)
    wb = _bf16_weights(eng.src_weights)
    units = ak.shard_units(ocfg, phi, rank)[1]
    heads = list(eng.heads)
    qn_h = qn.double().cpu().numpy()
    qr_h = qr.double().cpu().numpy()[..., :cfg.d_h_rope]
    alpha = ak.calib_alphas(ocfg)[2] if cfg.variant == "mlra" else 1.0
    errs = []
    for s in (seqs if seqs is not None else range(batch)):
        q_nope = np.zeros((cfg.h, cfg.d_h))
        q_rope = np.zeros((cfg.h, cfg.d_h_rope))
        q_nope[heads], q_rope[heads] = qn_h[s], qr_h[s]
        contribs = ak.attend_latent(ocfg, wb, ak.Cache(_streams(eng, s)), q_nope, q_rope, units)
        want = np.zeros((cfg.h, cfg.d_h))
        for head, vec in contribs:
            want[head] += vec
        want = alpha * want[heads]
        errs.append(ak.max_rel_err(want, got[s]))
    case = f"{variant}{'' if cfg.h == 24 else f'_h{cfg.h}'}_tp{phi}_rank{rank}_b{batch}_n{ctx}"
    _log(case, errs, {"nsplit": eng.nsplit, "page_size": eng.cache.page_size})
    assert max(errs) <= TOL, (case, errs)
    return eng


def test_configs1_tp1_b16_32k():
    """BASELINE configs[1] -- the N=1 bench workload: TP1, B = 16, 32K, nsplit 9, page 128."""
    eng = _check_latent("mlra4", 1, 0, 16, 32768)
    assert eng.nsplit == 9 and eng.cache.page_size == 128


@pytest.mark.parametrize("rank", [0, 3])
def test_headline_tp4_rank_b16_32k(rank):
    """The metric's own configuration: one TP4 rank (latent block k + rope), B = 16, 32K."""
    eng = _check_latent("mlra4", 4, rank, 16, 32768)
    assert eng.nsplit == 9


def test_configs2_tp4_rank_b16_64k():
    """BASELINE configs[2] shape per GPU: TP4 rank, B = 16, 64K."""
    _check_latent("mlra4", 4, 1, 16, 65536)


@pytest.mark.parametrize("phi,ctx", [(4, 131072), (1, 32768)])
def test_long_context_batch1(phi, ctx):
    """Batch 1 (the paper's decode regime): 148 splits of one sequence; K3 is the one-round-trip
    split merge + head GEMM (the split-K cluster grid, 24 heads x 8, exceeds one wave)."""
    eng = _check_latent("mlra4", phi, 0, 1, ctx)
    assert eng.nsplit == 148


@pytest.mark.parametrize("variant", ["mlra4", "mla"])
def test_paper_shape_64_heads_batch1(variant):
    """The paper's decode-benchmark shape (64 heads) on a TP4 rank, B = 1, 128K --
    the first point of the 64-head sweep (profiles/r2_sweep_h64_b1_long.md). MLRA-4 runs K2 with
    64-head groups and the merge + head GEMM K3 released at K2's epilogue."""
    from paper_2603_02188_b200.config import table_context

    eng = _check_latent(variant, 4, 0, 1, 131072, cfg=table_context()[variant])
    assert eng.nsplit == 148


@pytest.mark.parametrize("phi,rank", [(4, 2), (1, 0)])
def test_mla_comparison_rows(phi, rank):
    """vs_mla rows: MLA TP4 heads-sharded rank (6 heads, full latent) and MLA TP1, B = 16, 32K."""
    _check_latent("mla", phi, rank, 16, 32768, seqs=range(0, 16, 3))


@pytest.mark.parametrize("variant,phi", [("mlra2", 4), ("gla2", 2)])
def test_latent_variant_rows(variant, phi):
    """latent_variants rows: MLRA-2 TP4 rank and GLA-2 TP2 rank, B = 16, 32K."""
    _check_latent(variant, phi, 0, 16, 32768, seqs=range(0, 16, 5))


@pytest.mark.parametrize("phi", [1, 2])
def test_gqa_comparison_rows(phi):
    """vs_gqa rows: GQA (g = 6) TP1 and TP2 rank, B = 16, 32K."""
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.tp import shard_ownership

    bench = _bench()
    cfg = trained_config("gqa")
    own = shard_ownership(cfg, phi, 0) if phi > 1 else None
    eng, q = bench.make_gqa_engine(cfg, own, 16, 32768, 2000, torch.device("cuda", 0))
    got = eng.decode_attention(q).double().cpu().numpy()
    ocfg = ak.cfg_from(cfg)
    heads = list(eng.heads)
    slots = list(eng.own.kv_slots)
    qh = q.double().cpu().numpy()  # [B, G, R, dhp]
    errs = []
    for s in range(0, 16, 3):
        qq = np.zeros((cfg.h, cfg.d_h))
        qq[heads] = qh[s].reshape(len(heads), -1)[:, :cfg.d_h]
        streams = {"k": eng.cache.stream(s, "k").double().cpu().numpy(),
                   "v": eng.cache.stream(s, "v").double().cpu().numpy()}
        contribs = ak.attend_gqa(ocfg, ak.Cache(streams), qq, heads, slots)
        want = np.stack([vec for _, vec in contribs])
        errs.append(ak.max_rel_err(want, got[s]))
    _log(f"gqa_tp{phi}_rank0_b16_n32768", errs, {"nsplit": eng.nsplit})
    assert max(errs) <= TOL
