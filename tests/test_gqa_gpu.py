"""GPU parity of the GQA comparison variant (K2 GQA instantiation + split merge, through the
C ABI) against the CPU oracle's attend_gqa (attnkit/decode.py:232-240) and the reference's
golden outputs (tests/golden/p_gqa.npz). Tolerances as in test_decode_gpu.py."""

import numpy as np
import pytest
import torch

from golden_util import load, regen
from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu

TOL = 1e-2
TOL_REF = 2e-2
TOL_ORDER = 1e-3


def _mods():
    import paper_2603_02188_b200 as mlra
    from paper_2603_02188_b200 import gqa

    return mlra, gqa


def _fill(eng, seq_kv):
    """seq_kv: list of (k [n, g_local, d_h], v [n, g_local, d_h]) float64 -> bf16-rounded copies."""
    lay = eng.layout
    nmax = max(k.shape[0] for k, _ in seq_kv)
    rows = torch.zeros((len(seq_kv), nmax, lay.width), dtype=torch.bfloat16, device=eng.device)
    rounded = []
    for i, (k, v) in enumerate(seq_kv):
        kb, vb = ak.bf16_round(k), ak.bf16_round(v)
        rounded.append((kb, vb))
        rows[i, : k.shape[0]] = lay.pack_rows({"k": kb, "v": vb}, device=eng.device)
    eng.cache.fill(rows, [k.shape[0] for k, _ in seq_kv])
    return rounded


def _oracle(ocfg, k, v, q, heads, slots):
    cache = ak.Cache({"k": k, "v": v})
    out = np.zeros((len(heads), ocfg.d_h))
    for j, (head, vec) in enumerate(ak.attend_gqa(ocfg, cache, q, heads, slots)):
        out[j] = vec
    return out


def test_gqa_matches_oracle_and_reference_golden():
    mlra, gqa = _mods()
    meta, arrays = load("p_gqa")
    ocfg, w, hidden = regen(meta)
    cfg = mlra.AttnConfig(**meta["cfg"])
    n = meta["n"]
    # the golden step appends token n-1 and attends over all n tokens
    q, k, v = ak.gqa_projections(ocfg, w, hidden, range(n))
    eng = gqa.GqaDecodeEngine(cfg, batch=1, max_tokens=n, page_size=64)
    (kb, vb), = _fill(eng, [(k, v)])
    qb = ak.bf16_round(q[-1])
    got = eng.decode_attention(eng.prepare_queries(qb[None])).double().cpu().numpy()[0]
    want = _oracle(ocfg, kb, vb, qb, range(cfg.h), range(cfg.g))
    assert ak.max_rel_err(want, got) <= TOL
    assert ak.max_rel_err(arrays["out_absorbed"], got) <= TOL_REF


@pytest.mark.parametrize("page_size", [64, 128])
def test_gqa_ragged_batch_random_pages(page_size):
    """Ragged lengths across tile and page edges, a permuted page table, 2.9B GQA (g=6)."""
    mlra, gqa = _mods()
    cfg = mlra.trained_config("gqa").with_(d=256)
    ocfg = ak.cfg_from(cfg)
    lens = [1, 63, 64, 65, 127, 129, 1000, 2049]
    rng = np.random.default_rng(11)
    seq_kv, qs = [], []
    for n in lens:
        seq_kv.append((rng.standard_normal((n, cfg.g, cfg.d_h)), rng.standard_normal((n, cfg.g, cfg.d_h))))
        qs.append(ak.bf16_round(rng.standard_normal((cfg.h, cfg.d_h)) * 1.5))
    max_tok = max(lens)
    pages = -(-max_tok // page_size) * len(lens)
    order = torch.randperm(pages, generator=torch.Generator().manual_seed(3))
    eng = gqa.GqaDecodeEngine(cfg, batch=len(lens), max_tokens=max_tok, page_size=page_size, page_order=order)
    rounded = _fill(eng, seq_kv)
    got = eng.decode_attention(eng.prepare_queries(np.stack(qs))).double().cpu().numpy()
    for i in range(len(lens)):
        want = _oracle(ocfg, *rounded[i], qs[i], range(cfg.h), range(cfg.g))
        assert ak.max_rel_err(want, got[i]) <= TOL, f"sequence {i} (n={lens[i]})"


@pytest.mark.parametrize("phi", [2])
def test_gqa_tp_shards_assemble_full_output(phi):
    """tpsim.py sharding for gqa: each device holds g/phi KV heads and their query heads; the
    disjoint shard outputs concatenate to the single-device output (same kernels)."""
    mlra, gqa = _mods()
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = mlra.trained_config("gqa").with_(d=256)
    rng = np.random.default_rng(5)
    n = 1500
    k, v = rng.standard_normal((n, cfg.g, cfg.d_h)), rng.standard_normal((n, cfg.g, cfg.d_h))
    q = ak.bf16_round(rng.standard_normal((2, cfg.h, cfg.d_h)))
    full = gqa.GqaDecodeEngine(cfg, batch=2, max_tokens=n)
    _fill(full, [(k, v), (k[:700], v[:700])])
    ref = full.decode_attention(full.prepare_queries(q)).double().cpu().numpy()
    for dev in range(phi):
        own = shard_ownership(cfg, phi, dev)
        eng = gqa.GqaDecodeEngine(cfg, own, batch=2, max_tokens=n)
        slots = list(own.kv_slots)
        _fill(eng, [(k[:, slots], v[:, slots]), (k[:700, slots], v[:700, slots])])
        got = eng.decode_attention(eng.prepare_queries(q)).double().cpu().numpy()
        assert ak.max_rel_err(ref[:, list(own.heads)], got) <= TOL_ORDER


def test_gqa_kimi_context_shape():
    """Kimi context shape (table_context: h=64, g=8 -> 8 query heads per KV head), 4K tokens."""
    mlra, gqa = _mods()
    from paper_2603_02188_b200.config import table_context

    cfg = table_context()["gqa"].with_(d=256)
    ocfg = ak.cfg_from(cfg)
    rng = np.random.default_rng(9)
    n = 4096
    k, v = rng.standard_normal((n, cfg.g, cfg.d_h)), rng.standard_normal((n, cfg.g, cfg.d_h))
    q = ak.bf16_round(rng.standard_normal((cfg.h, cfg.d_h)))
    eng = gqa.GqaDecodeEngine(cfg, batch=1, max_tokens=n)
    (kb, vb), = _fill(eng, [(k, v)])
    got = eng.decode_attention(eng.prepare_queries(q[None])).double().cpu().numpy()[0]
    assert ak.max_rel_err(_oracle(ocfg, kb, vb, q, range(cfg.h), range(cfg.g)), got) <= TOL


def test_gqa_drop_in_step_and_sim_decode():
    """decode.absorbed_decode_step / tp.sim_decode for gqa against the oracle's step (same
    projections), with the reference's read accounting and the TP2 ledger ("6" d_h per token
    per device, golden p_gqa meta)."""
    mlra, gqa = _mods()
    from paper_2603_02188_b200 import decode, tp

    meta, arrays = load("p_gqa")
    ocfg, w, hidden = regen(meta)
    cfg = mlra.AttnConfig(**meta["cfg"])
    n = meta["n"]
    cache = decode.new_cache(cfg)
    q, k, v = ak.gqa_projections(ocfg, w, hidden[: n - 1], range(n - 1))
    for t in range(n - 1):
        cache.append({"k": k[t], "v": v[t]})
    cache.reads = 0
    out, cache = decode.absorbed_decode_step(cfg, w, cache, hidden[n - 1])
    assert ak.max_rel_err(arrays["out_absorbed"], out) <= TOL_REF
    assert cache.reads == meta["reads_after_step"]
    shards = tp.make_shards(cfg, w, 2)
    for t in range(n - 1):
        for s in shards:
            slots = list(s.own.kv_slots)
            s.cache.append({"k": k[t][slots], "v": v[t][slots]})
    out2, ledger = tp.sim_decode(shards, hidden[n - 1])
    assert ak.max_rel_err(arrays["out_tp2"], out2) <= TOL_REF
    assert ledger.to_json_dict()["per_token_load_dh"] == meta["tp"]["2"]["ledger"]
