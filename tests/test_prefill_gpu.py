"""Causal prefill into the paged cache (attnkit/latent.py:172-230) on
the GPU: outputs against the reference's own latent_prefill (golden vectors: first and last
4 tokens), the cache it leaves against the oracle's latent streams (bf16 rounding), and a
decode step continuing from it against the reference decode output (out_absorbed, which the
golden generator computes after a cache of the same n-1 tokens).

Tolerance: the decode kernels' (bf16 cache and queries, fp32 softmax / merge): max_rel_err
against the float64 reference <= 2e-2, the same gate as the decode parity tests."""

import numpy as np
import pytest
import torch

from oracle import attnkit_port as ak

from golden_util import load, regen

pytestmark = pytest.mark.gpu
CASES = ("refdims_mlra4", "refdims_mla", "refdims_mlra2", "refdims_gla2", "tiny_mlra4", "p_mlra4", "p_mla")


def _cfg(meta):
    import paper_2603_02188_b200 as mlra

    c = meta["cfg"]
    return mlra.AttnConfig(c["variant"], h=c["h"], d=c["d"], d_h=c["d_h"], d_h_rope=c["d_h_rope"], d_c=c["d_c"],
                           d_cq=c["d_cq"], g=c["g"], branches=c["branches"], scaling=c["scaling"])


@pytest.mark.parametrize("name", CASES)
def test_prefill_matches_reference_and_continues_decoding(name):
    import paper_2603_02188_b200 as mlra

    meta, arr = load(name)
    ocfg, w, hidden = regen(meta)
    cfg = _cfg(meta)
    n = meta["n"] - 1
    res = mlra.latent_prefill(cfg, w, hidden[:n], device="cuda:0")
    out = res.out
    assert out.shape == (n, cfg.h, cfg.d_h)
    for got, want, which in ((out[:4], arr["prefill_head"], "head"), (out[-4:], arr["prefill_tail"], "tail")):
        err = ak.max_rel_err(got, want)
        assert err <= 2e-2, f"{name} prefill {which}: max_rel_err {err:.3e}"
    # the cache it wrote holds the oracle's streams (bf16)
    streams = ak.latent_streams(ocfg, w, hidden[:n])
    cache = res.cache
    assert cache.n == n and cache.reads == 0
    for sname, want in streams.items():
        got = cache.peek(sname)
        scale = max(np.abs(want).max(), 1e-30)
        assert np.abs(got - want).max() / scale <= 2 ** -7, f"{name} stream {sname}"
    # decoding continues from the prefilled cache
    step, cache = mlra.absorbed_decode_step(cfg, w, cache, hidden[n])
    err = ak.max_rel_err(step, arr["out_absorbed"])
    assert err <= 2e-2, f"{name} decode after prefill: {err:.3e}"


def test_prefill_is_chunked_and_matches_decode_steps():
    """More queries than one kernel pass (PREFILL_CHUNK patched small) and a position offset:
    the prefill outputs equal the per-token decode outputs of the same tokens (the reference's
    tests/test_decode.py:83-94). Same kernels and bf16 weights on both sides; the prefill's n-row
    projections run as cuBLAS bf16 GEMMs (bf16 activations) and the decode's through K-1
    (fp32-split activations), so the two agree to the bf16 level, not bit for bit."""
    import paper_2603_02188_b200 as mlra
    from paper_2603_02188_b200 import decode as dec

    meta, _ = load("refdims_mlra4")
    ocfg, w, _ = regen(meta)
    cfg = _cfg(meta)
    rng = np.random.default_rng(0)
    hidden = rng.standard_normal((40, cfg.d))
    old = dec.PREFILL_CHUNK
    dec.PREFILL_CHUNK = 16
    try:
        res = mlra.latent_prefill(cfg, w, hidden, pos_offset=11, device="cuda:0")
    finally:
        dec.PREFILL_CHUNK = old
    cache = mlra.new_cache(cfg, pos_offset=11, device="cuda:0")
    for t in range(40):
        o, cache = mlra.absorbed_decode_step(cfg, w, cache, hidden[t])
        assert ak.max_rel_err(o, res.out[t]) <= 1e-2, t


def test_prefill_rejects_zoo_variants_and_empty_input():
    import paper_2603_02188_b200 as mlra

    cfg = mlra.trained_config("gqa")
    with pytest.raises(mlra.RoutingError):
        mlra.latent_prefill(cfg, {}, np.zeros((2, cfg.d)), device="cuda:0")
    meta, _ = load("refdims_mla")
    _, w, _ = regen(meta)
    res = mlra.latent_prefill(_cfg(meta), w, np.zeros((0, 32)), device="cuda:0")
    assert res.out.shape == (0, 4, 8) and res.cache.n == 0


@pytest.mark.parametrize("variant,n", [("mlra4", 1), ("mlra4", 129), ("mlra4", 1000), ("mlra2", 300), ("tiny", 700),
                                       ("mlra4", 4096)])
def test_prefill_kernel_matches_pseudo_sequence_path(variant, n):
    """K6 (tcgen05 causal prefill: 128 queries x one head per CTA, all branches and W^UV in-kernel)
    against the decode kernels run as n pseudo-sequences of lengths 1..n over the same cache --
    two independent implementations of latent.py:172-230 on the same bf16 cache and queries.
    Covers ragged tails (n % 128 != 0), the diagonal mask and the 2.9B / tiny geometries."""
    import paper_2603_02188_b200 as mlra
    from paper_2603_02188_b200 import decode as dec
    from paper_2603_02188_b200.config import trained_config
    from paper_2603_02188_b200.weights import weight_shapes

    cfg = mlra.tiny_config() if variant == "tiny" else trained_config(variant)
    rng = np.random.default_rng(n)
    w = {name: rng.standard_normal(shape) * 0.02 for name, shape in weight_shapes(cfg).items()}
    dev = torch.device("cuda", 0)
    st = dec._state(cfg, w, dev)
    h = torch.randn((n, cfg.d), generator=torch.Generator(device=dev).manual_seed(n), device=dev)
    outs = []
    for force in (False, True):
        cache = dec.new_cache(cfg, device=dev, initial_tokens=max(n, 128))
        assert dec.prefill_kernel_fits(cfg, cache.layout, st.own, cache.paged.page_size)
        outs.append(dec.prefill_into(cfg, st, cache, h, force_pseudo=force).double().cpu().numpy())
    errs = [ak.max_rel_err(outs[1][t], outs[0][t]) for t in range(n)]
    print(variant, n, "max_rel_err K6 vs pseudo-sequences", max(errs))
    # same bf16 cache and q~; the rotary query is rounded once (K6: scaled in the projection
    # epilogue) vs twice (pseudo path: rounded, then scaled by K1) -- one bf16 ulp apart
    assert max(errs) <= 1e-2, (int(np.argmax(errs)), max(errs))
