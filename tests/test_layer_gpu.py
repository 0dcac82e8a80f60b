"""DecodeEngine.decode_layer -- the attention layer from the new tokens' hidden rows (K-1 down ->
K0 append -> K-1 query -> [K1] -> K2 -> K3) against the oracle's latent_projections +
attend_local + reduce_contributions (attnkit/latent.py:129-159, decode.py:204-285) on the same
bf16 weights and the cache rows exactly as stored (prefix and the appended row).

Covers the pre-absorbed query (TP4 rank: W^UQ.W^UK_b pre-multiplied, K1 skipped) and the K1
path (TP1), graph replay, and the appended row against the reference's latent row."""

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


@pytest.mark.parametrize("variant,phi,rank", [("mlra4", 4, 2), ("mlra4", 1, 0), ("mlra2", 4, 1), ("mla", 1, 0)])
def test_decode_layer_matches_oracle(variant, phi, rank):
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = trained_config(variant)
    own = shard_ownership(cfg, phi, rank) if phi > 1 else None
    dev = torch.device("cuda", 0)
    B, ctx = 5, 700
    eng, hidden = _bench().make_layer_engine(cfg, own, B, ctx, 3, dev)
    kp = eng.kernel_projector(None)
    assert kp.absorbed == (variant in ("mlra4", "mlra2") and phi == 4)
    out = eng.decode_layer(hidden).double().cpu().numpy()
    assert eng.cache.seqlens.tolist() == [ctx + 1] * B
    ocfg = ak.cfg_from(cfg)
    wb = {k: ak.bf16_round(v) for k, v in eng.src_weights.items()}
    x = hidden.double().cpu().numpy()
    q_nope, q_rope, k_rope, latents = ak.latent_projections(ocfg, wb, x, [ctx] * B)
    units = ak.shard_units(ocfg, phi, rank)[1]
    heads = list(eng.heads)
    alpha = ak.calib_alphas(ocfg)[2] if cfg.variant == "mlra" else 1.0
    errs, row_errs = [], []
    for s in range(B):
        streams = {n: eng.cache.stream(s, n).double().cpu().numpy() for n in list(eng.layout.units) + ["rope"]}
        # the appended row (K0 on K-1's raw projections) vs the reference's latent rows
        row_errs.append(ak.max_rel_err(k_rope[s], streams["rope"][ctx]))
        for n in eng.layout.units:
            row_errs.append(ak.max_rel_err(latents[n][s], streams[n][ctx]))
        contribs = ak.attend_latent(ocfg, wb, ak.Cache(streams), q_nope[s], q_rope[s], units)
        want = np.zeros((cfg.h, cfg.d_h))
        for head, vec in contribs:
            want[head] += vec
        errs.append(ak.max_rel_err(alpha * want[heads], out[s]))
    print(variant, phi, "max_rel_err", max(errs), "row", max(row_errs))
    assert max(row_errs) <= 1e-2, row_errs
    assert max(errs) <= TOL, errs


def test_decode_layer_graph_replay_and_growth():
    """Captured in a CUDA graph: each replay appends one token per sequence (positions advance
    in-kernel) and equals the eager call on an identical engine."""
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = trained_config("mlra4")
    own = shard_ownership(cfg, 4, 0)
    dev = torch.device("cuda", 0)
    bench = _bench()
    a, ha = bench.make_layer_engine(cfg, own, 4, 300, 9, dev)
    b, hb = bench.make_layer_engine(cfg, own, 4, 300, 9, dev)
    eager = [a.decode_layer(ha).clone() for _ in range(3)]
    b.decode_layer(hb)  # warm (tensor maps, projector packs)
    b.cache.seqlens.fill_(300)
    res = torch.empty_like(eager[0])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        b.decode_layer(hb, out=res)
    b.cache.seqlens.fill_(300)
    for i in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(res, eager[i]), i
    assert b.cache.seqlens.tolist() == [303] * 4
