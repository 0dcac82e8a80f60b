"""Ragged batches (SURVEY.md 2.4 "K4" split scheduler, include/mlra_b200.h mlra_decode_plan): the
device-side plan's work table and the planned step against the oracle and the uniform-split step,
for sequences of very different lengths (attnkit/decode.py:204-230 decodes any length)."""

import os
import sys

import numpy as np
import pytest
import torch

from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LENS = [1, 100, 129, 1000, 5000, 20000, 127, 64000]


def _bench():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import bench

    return bench


def _engine(ragged, variant="mlra4", phi=4, lens=LENS, seed=5):
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = trained_config(variant)
    own = shard_ownership(cfg, phi, 1) if phi > 1 else None
    eng, qn, qr = _bench().make_engine(cfg, own, len(lens), max(lens), seed, torch.device("cuda", 0), ragged=ragged)
    eng.cache.seqlens.copy_(torch.tensor(lens, dtype=torch.int32))
    eng.cache._host_lens = list(lens)
    return cfg, own, eng, qn, qr


def test_plan_covers_every_tile_once():
    """The plan: every sequence's tiles exactly once, in ascending (sequence, split) order, at most
    ctas items, a balanced tile budget, empty slots marked -inf; deterministic."""
    from paper_2603_02188_b200 import _lib

    lens = [0, 1, 128, 129, 5000, 64000, 300, 70000, 1, 2]
    B, T, ctas, nmax, NB, H = len(lens), 128, 148, 64, 1, 24
    dev = torch.device("cuda", 0)
    sl = torch.tensor(lens, dtype=torch.int32, device=dev)
    plans = []
    for _ in range(2):
        plan = torch.full((ctas, 4), -7, dtype=torch.int32, device=dev)
        ns = torch.zeros(B, dtype=torch.int32, device=dev)
        lse = torch.zeros((B, nmax, NB, H), dtype=torch.float32, device=dev)
        rc = _lib.load().mlra_decode_plan(sl.data_ptr(), B, T, ctas, nmax, plan.data_ptr(), ns.data_ptr(),
                                          lse.data_ptr(), NB, H, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        plans.append((plan.cpu().numpy(), ns.cpu().numpy(), lse.cpu().numpy()))
    assert all((a == b).all() for a, b in zip(plans[0][:2], plans[1][:2]))
    plan, ns, lse = plans[0]
    tiles = [(n + T - 1) // T for n in lens]
    items = [tuple(r) for r in plan if r[0] >= 0]
    assert len(items) == int(ns.sum()) <= ctas
    assert all(r[0] == -1 for r in plan[len(items):])
    assert [(s, j) for s, j, _, _ in items] == sorted((s, j) for s, j, _, _ in items)
    budget = max(r[3] for r in items)
    assert budget <= max(-(-sum(tiles) // ctas), 1) * 2 + 1  # balanced: near total / ctas
    for s in range(B):
        mine = [r for r in items if r[0] == s]
        assert len(mine) == ns[s] >= 1
        covered = []
        for _, j, t0, n in mine:
            covered.extend(range(t0, t0 + n))
        assert covered == list(range(tiles[s])), s



@pytest.mark.parametrize("variant,phi", [("mlra4", 4), ("mlra4", 1), ("mla", 4)])
def test_ragged_step_matches_oracle_and_uniform(variant, phi):
    cfg, own, eng, qn, qr = _engine(True, variant, phi)
    _, _, ueng, _, _ = _engine(False, variant, phi)
    got = eng.decode_attention(qn, qr).double().cpu().numpy()
    uni = ueng.decode_attention(qn, qr).double().cpu().numpy()
    eng.check_numeric()
    ocfg = ak.cfg_from(cfg)
    wb = {k: ak.bf16_round(v) for k, v in eng.src_weights.items()}
    units = ak.shard_units(ocfg, phi, 1 if phi > 1 else 0)[1]
    heads = list(eng.heads)
    alpha = ak.calib_alphas(ocfg)[2] if cfg.variant == "mlra" else 1.0
    qn_h, qr_h = qn.double().cpu().numpy(), qr.double().cpu().numpy()[..., :cfg.d_h_rope]
    for s, n in enumerate(LENS):
        streams = {nm: eng.cache.stream(s, nm).double().cpu().numpy() for nm in list(eng.layout.units) + ["rope"]}
        assert streams["rope"].shape[0] == n
        q_nope = np.zeros((cfg.h, cfg.d_h))
        q_rope = np.zeros((cfg.h, cfg.d_h_rope))
        q_nope[heads], q_rope[heads] = qn_h[s], qr_h[s]
        want = np.zeros((cfg.h, cfg.d_h))
        for head, vec in ak.attend_latent(ocfg, wb, ak.Cache(streams), q_nope, q_rope, units):
            want[head] += vec
        want = alpha * want[heads]
        assert ak.max_rel_err(want, got[s]) <= 1e-2, (s, n)
        assert ak.max_rel_err(uni[s], got[s]) <= 5e-3, (s, n)  # other split boundaries: P rounds differently


def test_ragged_step_graph_replay():
    """The plan runs on the device: a captured step follows new lengths without re-capture."""
    cfg, own, eng, qn, qr = _engine(True)
    ref = eng.decode_attention(qn, qr).clone()
    g = torch.cuda.CUDAGraph()
    res = torch.empty_like(ref)
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        eng.decode_attention(qn, qr, out=res)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(res, ref)
    lens2 = [64000, 1, 3, 20000, 129, 5000, 1000, 100]
    eng.cache.seqlens.copy_(torch.tensor(lens2, dtype=torch.int32))
    g.replay()
    eager = eng.decode_attention(qn, qr)
    torch.cuda.synchronize()
    assert torch.equal(res, eager)
