"""The reference-side binding (integration/attnkit_b200.py, the module INTEGRATION.md describes as
attnkit/b200.py) driven by the UNMODIFIED reference package (attnkit installed in
baseline/_ref): attnkit's own cache, ownership, local_weights and token_queries feed the B200
library through ctypes, and the result is checked against the reference's golden outputs and
its own read accounting (tests/test_decode.py:34-44, :133-160 of the reference)."""

import os
import sys

import numpy as np
import pytest

from golden_util import load
from oracle import attnkit_port as ak

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TOL = 2e-2  # bf16 cache / queries on the GPU vs the float64 reference


def _attnkit():
    if os.path.isdir(REF) and REF not in sys.path:
        sys.path.append(REF)
    return pytest.importorskip("attnkit", reason="reference not installed in baseline/_ref")


def _binding():
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    try:
        import attnkit_b200
    finally:
        sys.path.pop(0)
    return attnkit_b200


def test_binding_signatures_match_the_header():
    """The binding declares the same ctypes signatures as the package's loader (which
    test_capi.py checks against include/mlra_b200.h), and every symbol resolves."""
    from paper_2603_02188_b200 import _lib, build

    b = _binding()
    for name, sig in b.SIGNATURES.items():
        assert _lib.SIGNATURES[name] == sig, name
    build.build()
    lib = b.load_library(_lib.LIB_PATH)
    for name in b.SIGNATURES:
        assert getattr(lib, name) is not None


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tiny_mlra4", "refdims_mla", "refdims_mlra4", "p_mlra4"])
def test_attnkit_step_through_binding(name):
    attnkit = _attnkit()
    from attnkit.decode import append_owned, full_ownership, token_cache_rows

    b = _binding()
    meta, arrays = load(name)
    cfg = attnkit.AttnConfig(**meta["cfg"])
    w = attnkit.build_weights(cfg, meta["sigma"], attnkit.Rng(meta["seed"]).split(*meta["w_path"]))
    n = meta["n"]
    hidden = attnkit.Rng(meta["seed"]).split(*meta["h_path"]).normal((n, cfg.d))
    cache = attnkit.new_cache(cfg)
    own = full_ownership(cfg)
    for t in range(n - 1):  # the prefix through attnkit's own append path
        append_owned(cfg, own, cache, token_cache_rows(cfg, w, hidden[t], t))
    cache.reads = 0
    out, cache = b.absorbed_decode_step(cfg, w, cache, hidden[n - 1])
    assert cache.n == n
    assert ak.max_rel_err(arrays["out_absorbed"], out) <= TOL
    assert cache.reads == meta["reads_after_step"]  # KvCache.read's charge, once per stream
    # the reference's own step on the same cache content agrees within the same tolerance
    ref_out, _ = attnkit.absorbed_decode_step(cfg, w, _copy_without_last(attnkit, cfg, cache), hidden[n - 1])
    assert ak.max_rel_err(ref_out, out) <= TOL


def _copy_without_last(attnkit, cfg, cache):
    from attnkit.cache import cache_from_streams

    streams = {k: np.asarray(cache.peek(k))[:-1] for k in cache.streams}
    return cache_from_streams(cfg, streams, cache.pos_offset)


@pytest.mark.gpu
def test_binding_routes_unserved_variants():
    attnkit = _attnkit()
    b = _binding()
    cfg = attnkit.AttnConfig("gqa", g=2, h=4, d=32, d_h=8)
    w = attnkit.build_weights(cfg, 0.3, attnkit.Rng(1).split("w"))
    with pytest.raises(attnkit.errors.RoutingError):
        b.absorbed_decode_step(cfg, w, attnkit.new_cache(cfg), np.zeros(cfg.d))
