"""The drop-in decode API (attnkit/decode.py, tpsim.py names) on the GPU, step by step,
against the oracle's restatement of the reference (and the reference's own golden outputs).
Structure follows the reference's tests/test_decode.py and tests/test_tpsim.py."""

from fractions import Fraction

import numpy as np
import pytest

from golden_util import load, regen
from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu

TOL = 2e-2  # GPU (bf16 cache/queries, fp32 projections) vs float64 reference


def _mlra():
    import paper_2603_02188_b200 as mlra

    return mlra


@pytest.mark.parametrize("name", ["tiny_mlra4", "refdims_mlra4", "refdims_mla", "p_mlra4", "p_mlra2", "p_gla2",
                                  "refdims_mlra2", "refdims_gla2"])
def test_decode_steps_track_reference(name):
    """absorbed_decode_step token by token from an empty cache; every step's output is
    compared with the oracle (f64) and the last one with the reference's golden output."""
    mlra = _mlra()
    meta, arrays = load(name)
    ocfg, w, hidden = regen(meta)
    cfg = mlra.AttnConfig(**meta["cfg"])
    n = meta["n"]
    steps = n if n <= 96 else 96
    start = n - steps
    ocache = ak.Cache(ak.latent_streams(ocfg, w, hidden[:start]) if start else {})
    cache = mlra.new_cache(cfg)
    if start:
        for t in range(start):  # prefix rows through the public append (one token at a time)
            cache.append({k: v[t] for k, v in ocache.streams.items()})
    for t in range(start, n):
        out, cache = mlra.absorbed_decode_step(cfg, w, cache, hidden[t])
        want = ak.absorbed_decode_step(ocfg, w, ocache, hidden[t])
        assert ak.max_rel_err(want, out) <= TOL, t
    assert cache.n == n
    assert ak.max_rel_err(arrays["out_absorbed"], out) <= TOL


@pytest.mark.parametrize("name", ["tiny_mlra4", "refdims_mla", "p_mlra4"])
def test_decode_step_naive_mode(name):
    """decode_step(mode="naive") (attnkit/decode.py:341-348 -> :309-338) returns the reference's
    materialised-KV result: the GPU evaluates it through absorption (equal in exact
    arithmetic), so it matches the golden out_naive within the bf16 tolerance, and the cache
    grows and is accounted like the absorbed step's."""
    mlra = _mlra()
    meta, arrays = load(name)
    ocfg, w, hidden = regen(meta)
    cfg = mlra.AttnConfig(**meta["cfg"])
    n = meta["n"]
    cache = mlra.new_cache(cfg)
    ocache = ak.Cache(ak.latent_streams(ocfg, w, hidden[: n - 1]))
    rows = cache.layout.pack_rows(ocache.streams, device="cuda:0")
    cache.paged.fill(rows[None], [n - 1])
    out, cache = mlra.decode_step(cfg, w, cache, hidden[n - 1], mode="naive")
    assert cache.n == n
    assert ak.max_rel_err(arrays["out_naive"], out) <= TOL
    with pytest.raises(mlra.errors.RoutingError):
        mlra.decode_step(cfg, w, cache, hidden[n - 1], mode="fused")


def test_read_accounting_and_append_only():
    """tests/test_decode.py:133-160: each step reads the whole state once; rows are frozen."""
    mlra = _mlra()
    cfg = mlra.AttnConfig("mla", h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16, scaling=True)
    w = mlra.build_weights(cfg, 0.3, mlra.Rng(38).split("w"))
    rng = mlra.Rng(38)
    cache = mlra.new_cache(cfg)
    assert cache.row_elements() == cfg.d_c + cfg.d_h_rope
    expected = 0
    for t in range(5):
        before = cache.reads
        mlra.absorbed_decode_step(cfg, w, cache, rng.split(f"h{t}").normal((cfg.d,)))
        assert cache.reads - before == (t + 1) * (cfg.d_c + cfg.d_h_rope)
        expected += (t + 1) * (cfg.d_c + cfg.d_h_rope)
    assert cache.reads == expected
    fp = cache.fingerprint(upto=2)
    mlra.absorbed_decode_step(cfg, w, cache, rng.split("h9").normal((cfg.d,)))
    assert cache.fingerprint(upto=2) == fp
    with pytest.raises(ValueError):
        cache.row("rope", 0)[0] = 1.0


def test_append_shape_errors():
    mlra = _mlra()
    cfg = mlra.tiny_config()
    cache = mlra.new_cache(cfg)
    with pytest.raises(mlra.ShapeMismatchError):
        cache.append({"rope": np.zeros(32)})
    rows = {f"latent_b{b}": np.zeros(64) for b in range(4)}
    rows["rope"] = np.zeros(31)
    with pytest.raises(mlra.ShapeMismatchError):
        cache.append(rows)
    with pytest.raises(mlra.ConfigError):
        cache.read("rope")  # empty stream (cache.py:62-63)


def test_attend_local_contributions_and_absorb_query():
    mlra = _mlra()
    from paper_2603_02188_b200.decode import attend_local, full_ownership, local_weights, reduce_contributions

    cfg = mlra.tiny_config()
    ocfg = ak.cfg_from(cfg)
    w = mlra.build_weights(cfg, 0.3, mlra.Rng(41))
    hidden = mlra.Rng(41).split("h").normal((9, cfg.d))
    cache = mlra.new_cache(cfg)
    streams = ak.latent_streams(ocfg, w.tensors, hidden)
    for t in range(9):
        cache.append({k: v[t] for k, v in streams.items()})
    qn, qr, _, _ = ak.latent_projections(ocfg, w.tensors, hidden[-1:], [8])
    own = full_ownership(cfg)
    contribs = attend_local(cfg, local_weights(cfg, w, own), own, cache, {"q_nope": qn[0], "q_rope": qr[0]})
    assert len(contribs) == 4 * cfg.h  # one per (head, branch)
    assert [h for h, _ in contribs[: cfg.h]] == list(range(cfg.h))
    out, kind = reduce_contributions(cfg, contribs)
    assert kind == "sum"
    want = ak.decode_attention(ocfg, w.tensors, streams, qn[0], qr[0])
    assert ak.max_rel_err(want, out) <= TOL
    # absorb_query vs the per-head loop (tests/test_decode.py:170-178)
    q = mlra.Rng(7).split("q").normal((4, 16))
    w_uk = mlra.Rng(7).split("w").normal((64, 4 * 16))
    got = mlra.absorb_query(q, w_uk)
    for i in range(4):
        ref = q[i] @ w_uk[:, i * 16:(i + 1) * 16].T
        assert np.max(np.abs(got[i] - ref)) <= 2e-2 * np.max(np.abs(ref))


@pytest.mark.parametrize("phi", [1, 2, 4, 8])
def test_sim_decode_matches_single_device_and_ledger(phi):
    """tests/test_tpsim.py:74-88 and :159-169 / :205-216 on the GPU path."""
    mlra = _mlra()
    cfg = mlra.tiny_config()
    w = mlra.build_weights(cfg, 0.25, mlra.Rng(100).split("w"))
    hidden = mlra.Rng(100).split("h").normal((4, cfg.d))
    ref_cache = mlra.new_cache(cfg)
    shards = mlra.make_shards(cfg, w, phi)
    for t in range(4):
        o_ref, _ = mlra.absorbed_decode_step(cfg, w, ref_cache, hidden[t])
        o_dist, ledger = mlra.sim_decode(shards, hidden[t])
        assert ak.max_rel_err(o_ref, o_dist) <= 1e-3
    per_token = {1: Fraction(9, 2), 2: Fraction(5, 2), 4: Fraction(3, 2), 8: Fraction(3, 2)}[phi]
    assert ledger.per_token_loads() == [per_token] * phi
    assert ledger.reduction == "sum"
    assert ledger.to_json_dict()["tp"] == phi
    if phi == 4:
        assert ledger.to_json_dict()["per_token_load_dh"] == ["1.5"] * 4
        assert ledger.replicated["rope"] == [0, 1, 2, 3]


def test_sim_decode_order_and_errors():
    mlra = _mlra()
    cfg = mlra.tiny_config()
    w = mlra.build_weights(cfg, 0.25, mlra.Rng(8).split("w"))
    hidden = mlra.Rng(8).split("h").normal((2, cfg.d))
    a, b = mlra.make_shards(cfg, w, 4), mlra.make_shards(cfg, w, 4)
    for t in range(2):
        o1, _ = mlra.sim_decode(a, hidden[t])
        o2, _ = mlra.sim_decode(b, hidden[t], order=[3, 1, 0, 2])
        assert np.array_equal(o1, o2)
    with pytest.raises(mlra.IntegrityError):
        mlra.sim_decode(a, hidden[0], order=[0, 0, 1, 2])
    with pytest.raises(mlra.ConfigError):
        mlra.make_shards(cfg, w, 16)


@pytest.mark.parametrize("name", ["refdims_mlra2", "refdims_gla2", "p_mlra2", "p_gla2"])
def test_grouped_latent_sim_decode_matches_reference(name):
    """MLRA-2 / GLA on the shared kernels under tpsim sharding: every TP degree the reference
    allows reproduces its golden output and per-device ledger."""
    mlra = _mlra()
    meta, arrays = load(name)
    ocfg, w, hidden = regen(meta)
    cfg = mlra.AttnConfig(**meta["cfg"])
    n = meta["n"]
    for phi_s, rec in meta["tp"].items():
        phi = int(phi_s)
        if "error" in rec:
            with pytest.raises(mlra.ConfigError):
                mlra.make_shards(cfg, w, phi)
            continue
        shards = mlra.make_shards(cfg, w, phi)
        out = ledger = None
        for t in range(n):
            out, ledger = mlra.sim_decode(shards, hidden[t])
        assert ak.max_rel_err(arrays[f"out_tp{phi}"], out) <= TOL, phi
        assert ledger.to_json_dict()["per_token_load_dh"] == rec["ledger"], phi
        assert ledger.reduction == rec["reduction"]
