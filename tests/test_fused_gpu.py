"""The fused single-launch decode step (fused_step.cuh, MLRA_FUSE_GRID) against the three-kernel
path and the oracle, its counter reset across launches / graph replays, and the numeric status
contract (attnkit/tensors.py:74-78: NaN in the logits or a row with no finite logit ->
NumericError). The fused step is an experiment compiled into K2 only with
-DMLRA_K2_FUSED_STEP (MLRA_NVCC_DEFS); its tests skip against the product library."""

import numpy as np
import pytest
import torch

from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _mlra():
    import paper_2603_02188_b200 as mlra

    return mlra


def _engine(cfg, w, lens, nsplit=None, own=None, page_size=128, seed=0):
    mlra = _mlra()
    ocfg = ak.cfg_from(cfg)
    eng = mlra.DecodeEngine(cfg, w, own, batch=len(lens), max_tokens=max(lens), page_size=page_size, nsplit=nsplit)
    rng = np.random.default_rng(seed)
    lay = eng.layout
    rows = torch.zeros((len(lens), max(lens), lay.width), dtype=torch.bfloat16, device=eng.device)
    streams = []
    for i, n in enumerate(lens):
        st = {u: ak.bf16_round(rng.standard_normal((n, lay.dl)) * 2.0) for u in lay.units}
        st["rope"] = ak.bf16_round(rng.standard_normal((n, lay.dr)))
        streams.append(st)
        rows[i, :n] = lay.pack_rows(st, device=eng.device)
    eng.cache.fill(rows, lens)
    qn = [ak.bf16_round(rng.standard_normal((cfg.h, cfg.d_h)) * 0.7) for _ in lens]
    qr = [ak.bf16_round(rng.standard_normal((cfg.h, cfg.d_h_rope))) for _ in lens]
    return eng, streams, qn, qr, ocfg


def _run(eng, qn, qr, out=None):
    from paper_2603_02188_b200.errors import ConfigError

    qn_t, qr_t = eng.prepare_queries(torch.tensor(np.stack(qn)), torch.tensor(np.stack(qr)))
    try:
        res = eng.decode_attention(qn_t, qr_t, out=out)
    except ConfigError as e:
        if "MLRA_K2_FUSED_STEP" in str(e):
            pytest.skip("library built without the fused-step experiment (-DMLRA_K2_FUSED_STEP)")
        raise
    torch.cuda.synchronize()
    return res.double().cpu().numpy()


@pytest.mark.parametrize("variant", ["mlra4", "mla", "mlra2", "gla2"])
def test_fused_step_matches_three_kernel_step(variant, monkeypatch):
    """Same inputs through the fused launch and through K1 -> K2 -> K3: the merge and
    up-projection arithmetic is the same (ascending splits, bf16 hi+lo, ascending chunks), so
    the results agree to fp32 rounding; both match the oracle."""
    monkeypatch.setenv("MLRA_FUSE_GRID", "1")
    mlra = _mlra()
    cfg = mlra.trained_config(variant).with_(d=256, d_cq=256)
    ocfg = ak.cfg_from(cfg)
    w = ak.build_weights(ocfg, 0.02, 21, ("w",))
    lens = [1, 100, 129, 3000, 4096, 777]
    eng, streams, qn, qr, ocfg = _engine(cfg, w, lens)
    fused = _run(eng, qn, qr)
    monkeypatch.setenv("MLRA_NO_FUSE", "1")
    plain = _run(eng, qn, qr)
    monkeypatch.delenv("MLRA_NO_FUSE")
    assert ak.max_rel_err(plain, fused) <= 1e-5
    wb = {k: ak.bf16_round(v) for k, v in w.items()}
    for i in range(len(lens)):
        want = ak.decode_attention(ocfg, wb, streams[i], qn[i], qr[i])
        assert ak.max_rel_err(want, fused[i]) <= TOL, (variant, i)


@pytest.mark.parametrize("batch,ctx", [(1, 20000), (16, 2048), (33, 1000), (64, 700)])
def test_fused_counters_reset_across_launches_and_graph_replays(batch, ctx, monkeypatch):
    """The last CTA resets the completion counters: back-to-back launches and CUDA-graph replays
    give bit-identical outputs (batch 33 / 64: several 16-sequence unit groups)."""
    monkeypatch.setenv("MLRA_FUSE_GRID", "1")
    mlra = _mlra()
    cfg = mlra.trained_config("mlra4").with_(d=256, d_cq=256)
    w = ak.build_weights(ak.cfg_from(cfg), 0.02, 22, ("w",))
    lens = [ctx - 7 * i for i in range(batch)]
    eng, streams, qn, qr, ocfg = _engine(cfg, w, lens, seed=batch)
    first = _run(eng, qn, qr)
    for _ in range(3):
        assert np.array_equal(first, _run(eng, qn, qr))
    qn_t, qr_t = eng.prepare_queries(torch.tensor(np.stack(qn)), torch.tensor(np.stack(qr)))
    out = torch.empty_like(eng.out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for _ in range(3):
            eng.decode_attention(qn_t, qr_t, out=out)
    for _ in range(4):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(first, out.double().cpu().numpy())
    assert int(eng.workspace.status.item()) == 0  # no numeric flag raised


def test_numeric_error_on_nan_in_cache():
    """A NaN cache row -> NaN logits -> NumericError on the drop-in path (tensors.py:74-75) and
    from DecodeEngine.check_numeric; a clean step afterwards passes."""
    mlra = _mlra()
    cfg = mlra.tiny_config()
    ocfg = ak.cfg_from(cfg)
    w = ak.build_weights(ocfg, 0.1, 23, ("w",))
    hidden = ak.normal(23, ("h",), (40, cfg.d))
    streams = ak.latent_streams(ocfg, w, hidden)
    # drop-in: attend_local over a cache holding one NaN
    cache = mlra.new_cache(cfg)
    bad = {k: v.copy() for k, v in streams.items()}
    bad["latent_b2"][17, 5] = np.nan
    cache.paged.fill(cache.layout.pack_rows(bad, device="cuda")[None], [40])
    qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [39])
    own = mlra.full_ownership(cfg)
    lw = mlra.local_weights(cfg, w, own)
    with pytest.raises(mlra.NumericError):
        mlra.attend_local(cfg, lw, own, cache, {"q_nope": qn[0], "q_rope": qr[0]})
    # the same cache with the row repaired is fine (the status word was reset by the check)
    cache.paged.fill(cache.layout.pack_rows(streams, device="cuda")[None], [40])
    contribs = mlra.attend_local(cfg, lw, own, cache, {"q_nope": qn[0], "q_rope": qr[0]})
    assert len(contribs) == 4 * cfg.h
    # serving engine: the step runs (no sync), check_numeric raises once, then clears
    eng, st, q1, q2, _ = _engine(cfg, w, [300, 64])
    eng.cache.pool[3, 7] = float("nan")
    _run(eng, q1, q2)
    with pytest.raises(mlra.NumericError):
        eng.check_numeric()
    eng.cache.pool[3, 7] = 0.0
    _run(eng, q1, q2)
    eng.check_numeric()


def test_numeric_error_gqa_and_no_finite_row():
    """GQA path: a NaN key -> NumericError. Latent path: an all -inf rotary key row set makes
    every logit -inf (no finite entry, tensors.py:76-77) -> NumericError."""
    mlra = _mlra()
    cfg = mlra.trained_config("gqa").with_(d=256)
    w = mlra.build_weights(cfg, 0.02, mlra.Rng(24).split("w"))
    cache = mlra.new_cache(cfg)
    rng = mlra.Rng(24)
    for t in range(20):
        mlra.absorbed_decode_step(cfg, w, cache, rng.split(f"h{t}").normal((cfg.d,)))
    cache.paged.pool[5, 3] = float("nan")
    with pytest.raises(mlra.NumericError):
        mlra.absorbed_decode_step(cfg, w, cache, rng.split("bad").normal((cfg.d,)))
    lat = mlra.trained_config("mla").with_(d=256, d_cq=256)
    eng, st, q1, q2, _ = _engine(lat, ak.build_weights(ak.cfg_from(lat), 0.02, 25, ("w",)), [200])
    lay = eng.layout
    eng.cache.pool[:, lay.nb * lay.dlp:] = float("-inf")  # rope keys -inf: q_rope . k = -inf everywhere
    q2 = [np.abs(q) + 0.5 for q in q2]
    _run(eng, q1, q2)
    with pytest.raises(mlra.NumericError):
        eng.check_numeric()
