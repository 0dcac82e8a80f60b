"""The oracle (oracle/attnkit_port.py) against golden vectors from the real reference."""

import numpy as np
import pytest

from oracle import attnkit_port as ak
from golden_util import CASES, load, regen


@pytest.mark.parametrize("name", CASES)
def test_inputs_regenerate_bit_exactly(name):
    meta, _ = load(name)
    cfg, w, hidden = regen(meta)
    assert ak.sha(hidden) == meta["sha_hidden"]
    for k, digest in meta["sha_w"].items():
        assert ak.sha(w[k]) == digest, k


@pytest.mark.parametrize("name", CASES)
def test_cache_rows_match_reference(name):
    meta, arrays = load(name)
    cfg, w, hidden = regen(meta)
    n = meta["n"]
    if cfg.variant == "gqa":
        q, k, v = ak.gqa_projections(cfg, w, hidden[: n - 1], range(n - 1))
        streams = {"k": k, "v": v}
    else:
        streams = ak.latent_streams(cfg, w, hidden[: n - 1])
    for k, digest in meta["sha_streams"].items():
        # sha over float64 bytes: the restated projections must be bitwise identical
        got = ak.sha(streams[k])
        if got != digest:  # allow last-ulp BLAS differences, but require 1e-14 agreement
            head = arrays.get(f"stream_{k}_head")
            assert head is not None and np.max(np.abs(streams[k][:4] - head)) < 1e-13
        if f"stream_{k}_head" in arrays:
            np.testing.assert_allclose(streams[k][:4], arrays[f"stream_{k}_head"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", CASES)
def test_absorbed_step_matches_reference(name):
    meta, arrays = load(name)
    cfg, w, hidden = regen(meta)
    n = meta["n"]
    cache = ak.Cache()
    if cfg.variant == "gqa":
        q, k, v = ak.gqa_projections(cfg, w, hidden[: n - 1], range(n - 1))
        cache.streams = {"k": k, "v": v}
    else:
        cache.streams = ak.latent_streams(cfg, w, hidden[: n - 1])
    out = ak.absorbed_decode_step(cfg, w, cache, hidden[n - 1])
    assert ak.max_rel_err(arrays["out_absorbed"], out) <= 1e-10
    assert cache.reads == meta["reads_after_step"]


@pytest.mark.parametrize("name", [c for c in CASES if c != "p_gqa"])
def test_naive_step_and_queries_match_reference(name):
    meta, arrays = load(name)
    cfg, w, hidden = regen(meta)
    n = meta["n"]
    cache = ak.Cache(ak.latent_streams(cfg, w, hidden[: n - 1]))
    out = ak.naive_decode_step(cfg, w, cache, hidden[n - 1])
    assert ak.max_rel_err(arrays["out_naive"], out) <= 1e-10
    q_nope, q_rope, _, _ = ak.latent_projections(cfg, w, hidden[n - 1:], [n - 1])
    np.testing.assert_allclose(q_nope[0], arrays["q_nope"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(q_rope[0], arrays["q_rope"], rtol=0, atol=1e-12)
    # absorbed over the complete cache == the attention-only entry the GPU path computes
    streams = ak.latent_streams(cfg, w, hidden)
    att = ak.decode_attention(cfg, w, streams, q_nope[0], q_rope[0])
    assert ak.max_rel_err(arrays["out_absorbed"], att) <= 1e-10


@pytest.mark.parametrize("name", [c for c in CASES if c in ("tiny_mlra4", "refdims_mlra4", "refdims_mla",
                                                           "refdims_mlra2", "refdims_gla2")])
def test_tensor_parallel_matches_reference(name):
    meta, arrays = load(name)
    cfg, w, hidden = regen(meta)
    n = meta["n"]
    streams = ak.latent_streams(cfg, w, hidden)
    q_nope, q_rope, _, _ = ak.latent_projections(cfg, w, hidden[n - 1:], [n - 1])
    for phi_s, rec in meta["tp"].items():
        phi = int(phi_s)
        if "error" in rec:
            with pytest.raises(ak.OracleError):
                ak.sim_decode_attention(cfg, w, streams, q_nope[0], q_rope[0], phi)
            continue
        out, kind, reads = ak.sim_decode_attention(cfg, w, streams, q_nope[0], q_rope[0], phi)
        assert ak.max_rel_err(arrays[f"out_tp{phi}"], out) <= 1e-10
        assert kind == rec["reduction"]
        assert reads == rec["reads_last"]
        # the reference ledger's per-token loads == the closed-form per-device load
        assert [ak.Fraction(x) for x in rec["ledger"]] == [ak.per_device_load(cfg, phi)] * phi


def test_per_device_load_table():
    p = ak.Cfg("mlra", 24, 3072, 128, 64, 512, 1024, branches=4, scaling=True)
    assert [str(ak.per_device_load(p, phi)) for phi in (1, 2, 4, 8)] == ["9/2", "5/2", "3/2", "3/2"]
    mla = ak.Cfg("mla", 24, 3072, 128, 64, 512, 1536, scaling=True)
    assert {ak.per_device_load(mla, phi) for phi in (1, 2, 4, 8)} == {ak.Fraction(9, 2)}
    # MLRA-2 also reaches 1.5 d_h at TP4; GLA-2 plateaus at 2.5 d_h
    m2 = ak.Cfg("mlra", 24, 3072, 128, 64, 512, 1024, branches=2, scaling=True)
    assert [str(ak.per_device_load(m2, phi)) for phi in (1, 2, 4, 8)] == ["9/2", "5/2", "3/2", "3/2"]
    g2 = ak.Cfg("gla", 24, 3072, 128, 64, 512, 1024, g=2, scaling=True)
    assert [str(ak.per_device_load(g2, phi)) for phi in (1, 2, 4, 8)] == ["9/2", "5/2", "5/2", "5/2"]


def test_softmax_guards():
    with pytest.raises(ak.OracleError):
        ak.softmax_rows(np.array([[np.nan, 1.0]]))
    with pytest.raises(ak.OracleError):
        ak.softmax_rows(np.array([[-np.inf, -np.inf]]))


def test_bf16_round_is_round_to_nearest_even():
    x = np.array([1.0, 1.0 + 2.0**-8, 1.0 + 3 * 2.0**-9, -2.5, 3.0e-3])
    r = ak.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0 + 2.0**-7 and r[3] == -2.5
    assert abs(r[4] - 3.0e-3) / 3.0e-3 < 2**-8
