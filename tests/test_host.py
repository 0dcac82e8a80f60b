"""Host-side logic of the product package (no GPU): config, seeded weights, cost formulas,
sharding rules, row layouts and weight packing."""

from fractions import Fraction

import numpy as np
import pytest

import paper_2603_02188_b200 as mlra
from golden_util import load
from oracle import attnkit_port as ak
from paper_2603_02188_b200.cache import RowLayout
from paper_2603_02188_b200.config import AttnConfig, trained_config
from paper_2603_02188_b200.errors import ConfigError, RoutingError


def test_config_defaults_and_validation():
    c = AttnConfig("mlra", branches=4, h=4, d=64, d_h=16, d_cq=32)
    assert (c.d_c, c.d_h_rope, c.block_dim) == (64, 8, 16)
    assert c.tau == pytest.approx((16 + 8) ** -0.5)
    with pytest.raises(ConfigError):
        AttnConfig("mlra", branches=3, h=4, d=64, d_h=16)
    with pytest.raises(ConfigError):
        AttnConfig("mlra", branches=4, h=3, d=64, d_h=16)
    with pytest.raises(ConfigError):
        AttnConfig("nope", h=4, d=64, d_h=16)
    p = trained_config("mlra4")
    assert (p.h, p.d_h, p.d_c, p.d_h_rope, p.d_cq) == (24, 128, 512, 64, 1024)
    assert p.tau == pytest.approx(1 / 192 ** 0.5)


def test_calib_factors():
    p = trained_config("mlra4")
    sf = mlra.calib_factors(p)
    assert sf.alpha_attn == pytest.approx(0.5)
    assert sf.alpha_kv == pytest.approx(24 ** 0.5)
    assert sf.alpha_q == pytest.approx(3 ** 0.5)
    assert mlra.calib_factors(trained_config("mla")).alpha_attn == 1.0


@pytest.mark.parametrize("name", ["tiny_mlra4", "p_mla", "p_gqa"])
def test_product_rng_and_weights_match_reference(name):
    meta, _ = load(name)
    cfg = AttnConfig(**meta["cfg"])
    w = mlra.build_weights(cfg, meta["sigma"], mlra.Rng(meta["seed"]).split(meta["w_path"][0]))
    for k, digest in meta["sha_w"].items():
        assert ak.sha(w[k]) == digest, k
    hidden = mlra.Rng(meta["seed"]).split(meta["h_path"][0]).normal((meta["n"], cfg.d))
    assert ak.sha(hidden) == meta["sha_hidden"]


def test_cost_formulas():
    p = trained_config("mlra4")
    assert [mlra.per_device_load(p, phi) for phi in (1, 2, 4, 8)] == [Fraction(9, 2), Fraction(5, 2),
                                                                      Fraction(3, 2), Fraction(3, 2)]
    assert mlra.algorithmic_bytes(p, 4, [32768] * 16) == 201326592
    assert mlra.algorithmic_bytes(p, 1, [32768] * 16) == 603979776
    assert mlra.algorithmic_bytes(trained_config("mla"), 4, [32768] * 16) == 603979776
    assert mlra.decode_flops_per_device(p, 4, 32768) * 16 == 16 * 24 * 32768 * (4 * 128 + 2 * 64)
    from paper_2603_02188_b200.costs import fraction_str

    assert [fraction_str(x) for x in (Fraction(3, 2), Fraction(1, 3), Fraction(4))] == ["1.5", "1/3", "4"]


def test_shard_ownership_rules():
    from paper_2603_02188_b200.tp import shard_ownership

    p = trained_config("mlra4")
    for k in range(4):
        own = shard_ownership(p, 4, k)
        assert [u.block for u in own.units] == [k] and own.heads == tuple(range(24))
    own = shard_ownership(p, 2, 1)
    assert [u.block for u in own.units] == [2, 3]
    own8 = [shard_ownership(p, 8, k) for k in range(8)]
    assert [o.units[0].block for o in own8] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert own8[1].heads == tuple(range(12, 24))
    mla = trained_config("mla")
    assert shard_ownership(mla, 4, 3).heads == tuple(range(18, 24))
    with pytest.raises(ConfigError, match="TP degree"):
        shard_ownership(p, 16, 0)
    with pytest.raises(RoutingError):
        shard_ownership(trained_config("mla").with_(variant="mha"), 2, 0)


@pytest.mark.parametrize("name", ["mlra2", "gla2", "gla4"])
@pytest.mark.parametrize("phi", [1, 2, 4, 8])
def test_grouped_latent_shard_ownership_matches_oracle(name, phi):
    """tpsim.py:58-131 for MLRA-2 and GLA (2.9B shapes): same heads and units as the oracle."""
    from oracle import attnkit_port as ak
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = trained_config(name)
    ocfg = ak.cfg_from(cfg)
    for k in range(phi):
        try:
            heads, units = ak.shard_units(ocfg, phi, k)
        except ak.OracleError:
            with pytest.raises(ConfigError):
                shard_ownership(cfg, phi, k)
            continue
        own = shard_ownership(cfg, phi, k)
        assert own.heads == tuple(heads)
        assert [(u.stream, u.group, u.block, u.heads) for u in own.units] == [tuple(u) for u in units]


def test_grouped_latent_kernel_geometry_and_packing():
    """MLRA-2 / GLA units with different head sets: block-diagonal packs on the shared kernels."""
    import torch

    from paper_2603_02188_b200.decode import full_ownership, kernel_geometry, local_weights, row_layout

    for name, geom in (("mlra2", (4, 128)), ("gla2", (1, 512)), ("gla4", (4, 128))):
        cfg = trained_config(name).with_(d=64)
        w = mlra.build_weights(cfg, 0.02, mlra.Rng(3))
        own = full_ownership(cfg)
        lay = row_layout(cfg, own)
        assert kernel_geometry(lay, own) == geom
        uk, uv = local_weights(cfg, w, own).packed(lay, torch.device("cpu"), own)
        assert tuple(uk.shape) == (24, 128, 512) and tuple(uv.shape) == (24, 512, 128)
        for i, u in enumerate(own.units):  # zero where the unit does not serve the head
            cols = slice(i * lay.dlp, (i + 1) * lay.dlp)
            others = [hd for hd in range(24) if hd not in u.heads]
            assert float(uk[others][:, :, cols].abs().max()) == 0.0
            assert float(uk[list(u.heads)][:, :, cols].abs().max()) > 0.0


@pytest.mark.parametrize("shape,phi", [("2.9b", 1), ("2.9b", 2), ("kimi", 1), ("kimi", 4), ("kimi", 8)])
def test_gqa_shard_ownership_matches_oracle(shape, phi):
    """tpsim.py:58-131 for gqa (g=6 at the 2.9B shape, g=8 at the Kimi context shape):
    KV-head axis, grouped heads."""
    from oracle import attnkit_port as ak
    from paper_2603_02188_b200.config import table_context
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = trained_config("gqa") if shape == "2.9b" else table_context()["gqa"]
    for k in range(phi):
        own = shard_ownership(cfg, phi, k)
        heads, slots = ak.shard_units(ak.cfg_from(cfg), phi, k)
        assert own.heads == tuple(heads) and own.kv_slots == tuple(slots) and own.units == ()


def test_gqa_layout_pack_and_extract():
    import torch

    from paper_2603_02188_b200.cache import GqaLayout

    lay = GqaLayout(3, 8)
    assert (lay.dhp, lay.width) == (64, 384) and lay.row_shapes() == {"k": (3, 8), "v": (3, 8)}
    k = np.arange(24, dtype=np.float64).reshape(3, 8)
    v = -np.arange(24, dtype=np.float64).reshape(3, 8) - 1
    row = lay.pack_rows({"k": k, "v": v}, device=torch.device("cpu"))
    assert row.shape == (384,)
    r = row.float().numpy()
    assert list(r[64:72]) == list(k[1]) and r[72:128].sum() == 0 and list(r[192 + 128:192 + 136]) == list(v[2])
    np.testing.assert_array_equal(lay.extract("k", row[None]).float().numpy()[0], k)
    np.testing.assert_array_equal(lay.extract("v", row[None]).float().numpy()[0], v)
    assert GqaLayout(6, 128).width == 1536
    with pytest.raises(ConfigError):
        GqaLayout(1, 256).dhp


def test_row_layout_padding():
    lay = RowLayout(tuple(f"latent_b{b}" for b in range(4)), 128, 64)
    assert (lay.dlp, lay.drp, lay.width, lay.geometry) == (128, 64, 576, (1, 128))
    tiny = RowLayout(tuple(f"latent_b{b}" for b in range(4)), 8, 4)
    assert (tiny.dlp, tiny.drp, tiny.width) == (64, 16, 272)
    mla = RowLayout(("latent",), 512, 64)
    assert mla.geometry == (4, 128) and mla.width == 576
    assert mla.column("rope") == slice(512, 576)
    with pytest.raises(ConfigError):
        RowLayout(("latent",), 512, 96).drp


def test_weight_pack_layout():
    import torch

    from paper_2603_02188_b200.decode import full_ownership, local_weights, row_layout

    cfg = AttnConfig("mlra", branches=4, h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16, scaling=True)
    w = mlra.build_weights(cfg, 0.3, mlra.Rng(1))
    own = full_ownership(cfg)
    lw = local_weights(cfg, w, own)
    lay = row_layout(cfg, own)
    uk, uv = lw.packed(lay, torch.device("cpu"))
    assert tuple(uk.shape) == (4, 8, 4 * 64) and tuple(uv.shape) == (4, 4 * 64, 8)
    bs = cfg.block_dim
    for b in range(4):
        ref = w["w_uk"][b * bs:(b + 1) * bs].reshape(bs, 4, 8)  # (lat, h, d_h)
        got = uk[:, :, b * 64:b * 64 + bs].float().numpy()      # (h, d_h, lat)
        np.testing.assert_allclose(got, np.transpose(ref, (1, 2, 0)), rtol=1e-2, atol=1e-2)
        assert float(uk[:, :, b * 64 + bs:(b + 1) * 64].abs().max()) == 0.0  # zero padding
        refv = w["w_uv"][b * bs:(b + 1) * bs].reshape(bs, 4, 8)
        np.testing.assert_allclose(uv[:, b * 64:b * 64 + bs, :].float().numpy(), np.transpose(refv, (1, 0, 2)),
                                   rtol=1e-2, atol=1e-2)


def test_pack_rows_places_streams():
    import torch

    lay = RowLayout(("latent_b0", "latent_b1"), 3, 2)
    rows = {"latent_b0": np.array([1.0, 2, 3]), "latent_b1": np.array([4.0, 5, 6]), "rope": np.array([7.0, 8])}
    out = lay.pack_rows(rows, device=torch.device("cpu")).float().numpy()
    assert out.shape == (2 * 64 + 16,)
    assert list(out[:3]) == [1, 2, 3] and list(out[64:67]) == [4, 5, 6] and list(out[128:130]) == [7, 8]
    assert out[3:64].sum() == 0 and out[130:].sum() == 0


def test_decode_routing_errors():
    from paper_2603_02188_b200.decode import decode_step, full_ownership

    own = full_ownership(trained_config("gqa"))
    assert own.kv_slots == tuple(range(6)) and own.heads == tuple(range(24))
    with pytest.raises(RoutingError):
        full_ownership(trained_config("mla").with_(variant="mha"))
    cfg = AttnConfig("mlra", branches=2, h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16)
    own = full_ownership(cfg)  # mlra-2: (group, block) units over half the heads each
    assert [(u.group, u.block, u.heads) for u in own.units] == [(0, 0, (0, 1)), (0, 1, (0, 1)), (1, 0, (2, 3)),
                                                                (1, 1, (2, 3))]
    with pytest.raises(RoutingError):
        full_ownership(trained_config("mla").with_(variant="tpa"))
    with pytest.raises(RoutingError):
        decode_step(trained_config("mlra4"), None, None, None, mode="turbo")
    with pytest.raises(RoutingError):  # naive covers the latent family only (decode.py:313-316)
        decode_step(trained_config("gqa"), None, None, None, mode="naive")


def test_step_state_cache_is_bounded():
    """The per-weight-set device state is an LRU (decode._STATE_MAX entries), not a leak."""
    from paper_2603_02188_b200 import decode as dec

    cfg = dec.AttnConfig("mlra", branches=4, h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16)
    saved = dict(dec._STATE)
    dec._STATE.clear()
    try:
        weights = [{"w_uk": np.zeros((32, 32)), "w_uv": np.zeros((32, 32))} for _ in range(dec._STATE_MAX + 3)]
        orig = dec._StepState

        class Dummy:
            def __init__(self, cfg, w, device):
                pass

        dec._StepState = Dummy
        try:
            for w in weights:
                dec._state(cfg, w, "cpu")
        finally:
            dec._StepState = orig
        assert len(dec._STATE) == dec._STATE_MAX
        assert [k[1] for k in dec._STATE] == [id(w) for w in weights[-dec._STATE_MAX:]]
    finally:
        dec._STATE.clear()
        dec._STATE.update(saved)
