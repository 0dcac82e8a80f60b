"""GPU parity of the B200 decode path (K0-K3 through the C ABI) against the CPU oracle.

Tolerance: max_rel_err <= 1e-2 against the float64 oracle evaluated
on the SAME bf16-rounded cache, weights and queries; <= 2e-2 against the reference's own
float64 outputs (which additionally see the bf16 rounding of the inputs); <= 1e-3 between
two GPU evaluations that differ only in reduction order (TP vs single device, split count).
"""

import numpy as np
import pytest
import torch

from golden_util import load, regen
from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu

TOL = 1e-2
TOL_REF = 2e-2
TOL_ORDER = 1e-3


def _mlra():
    import paper_2603_02188_b200 as mlra

    return mlra


def _bf16_weights(w):
    out = dict(w)
    for k in w:
        if k.startswith(("w_uk", "w_uv")):  # single latent or per-group up-projections
            out[k] = ak.bf16_round(w[k])
    return out


def _engine_inputs(engine, seq_streams):
    """Fill engine.cache with bf16-rounded streams of each sequence; returns rounded copies."""
    lay = engine.layout
    B = len(seq_streams)
    nmax = max(s["rope"].shape[0] for s in seq_streams)
    rows = torch.zeros((B, nmax, lay.width), dtype=torch.bfloat16, device=engine.device)
    rounded = []
    for i, st in enumerate(seq_streams):
        r = {k: ak.bf16_round(v) for k, v in st.items()}
        rounded.append(r)
        n = st["rope"].shape[0]
        rows[i, :n] = lay.pack_rows({k: r[k] for k in list(lay.units) + ["rope"]}, device=engine.device)
    engine.cache.fill(rows, [s["rope"].shape[0] for s in seq_streams])
    return rounded


def _run(engine, q_nope, q_rope):
    qn, qr = engine.prepare_queries(torch.tensor(np.stack(q_nope)), torch.tensor(np.stack(q_rope)))
    out = engine.decode_attention(qn, qr)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def _oracle_cfg(cfg):
    return ak.cfg_from(cfg)


@pytest.mark.parametrize("name", ["tiny_mlra4", "p_mlra4", "p_mla", "refdims_mlra4", "refdims_mla", "p_mlra2", "p_gla2",
                                  "refdims_mlra2", "refdims_gla2"])
def test_engine_matches_oracle_and_reference(name):
    mlra = _mlra()
    meta, arrays = load(name)
    ocfg, w, hidden = regen(meta)
    cfg = mlra.AttnConfig(**meta["cfg"])
    n = meta["n"]
    streams = ak.latent_streams(ocfg, w, hidden)
    q_nope = ak.bf16_round(arrays["q_nope"])
    q_rope = ak.bf16_round(arrays["q_rope"])
    eng = mlra.DecodeEngine(cfg, w, batch=1, max_tokens=n, page_size=64)
    rs = _engine_inputs(eng, [streams])[0]
    got = _run(eng, [q_nope], [q_rope])[0]
    want = ak.decode_attention(ocfg, _bf16_weights(w), rs, q_nope, q_rope)
    assert ak.max_rel_err(want, got) <= TOL
    assert ak.max_rel_err(arrays["out_absorbed"], got) <= TOL_REF


@pytest.mark.parametrize("variant", ["mlra", "mla"])
@pytest.mark.parametrize("page_size", [64, 128])
def test_ragged_batch_random_pages(variant, page_size):
    """Lengths straddling tile (64/128) and page boundaries, non-contiguous page tables."""
    mlra = _mlra()
    cfg = mlra.trained_config("mlra4" if variant == "mlra" else "mla").with_(d=256, d_cq=256)
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.02, 3, ("w",))
    lens = [1, 63, 64, 65, 127, 129, 1000, 2049]
    seq_streams, qns, qrs = [], [], []
    for i, n in enumerate(lens):
        hidden = ak.normal(3, ("h", i), (n, cfg.d))
        seq_streams.append(ak.latent_streams(ocfg, w, hidden))
        qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [n - 1])
        qns.append(ak.bf16_round(qn[0]))
        qrs.append(ak.bf16_round(qr[0]))
    maxp = -(-max(lens) // page_size)
    order = torch.randperm(len(lens) * maxp, generator=torch.Generator().manual_seed(5))
    eng = mlra.DecodeEngine(cfg, w, batch=len(lens), max_tokens=max(lens), page_size=page_size, page_order=order,
                            nsplit=3)
    rounded = _engine_inputs(eng, seq_streams)
    got = _run(eng, qns, qrs)
    wb = _bf16_weights(w)
    for i in range(len(lens)):
        want = ak.decode_attention(ocfg, wb, rounded[i], qns[i], qrs[i])
        assert ak.max_rel_err(want, got[i]) <= TOL, (i, lens[i])


def test_tensor_parallel_shards_sum_to_single_device():
    """MLRA-4 at TP 2/4/8: per-device engines (one latent block + the replicated rope per
    device at TP4) whose outputs, summed (the NCCL all-reduce), equal TP1 and the oracle."""
    mlra = _mlra()
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = mlra.trained_config("mlra4").with_(d=256, d_cq=256)
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.02, 4, ("w",))
    lens = [700, 1300]
    seq_streams, qns, qrs = [], [], []
    for i, n in enumerate(lens):
        hidden = ak.normal(4, ("h", i), (n, cfg.d))
        seq_streams.append(ak.latent_streams(ocfg, w, hidden))
        qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [n - 1])
        qns.append(ak.bf16_round(qn[0]))
        qrs.append(ak.bf16_round(qr[0]))
    full = mlra.DecodeEngine(cfg, w, batch=2, max_tokens=max(lens))
    rounded = _engine_inputs(full, seq_streams)
    ref1 = _run(full, qns, qrs)
    wb = _bf16_weights(w)
    for i in range(2):
        assert ak.max_rel_err(ak.decode_attention(ocfg, wb, rounded[i], qns[i], qrs[i]), ref1[i]) <= TOL
    for phi in (2, 4, 8):
        total = np.zeros_like(ref1)
        for k in range(phi):
            own = shard_ownership(cfg, phi, k)
            eng = mlra.DecodeEngine(cfg, w, own, batch=2, max_tokens=max(lens))
            _engine_inputs(eng, [{u: s[u] for u in list(eng.layout.units) + ["rope"]} for s in seq_streams])
            part = _run(eng, qns, qrs)
            total[:, list(own.heads)] += part
        assert ak.max_rel_err(ref1, total) <= TOL_ORDER, phi


def test_mla_heads_sharded_tp4():
    mlra = _mlra()
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = mlra.trained_config("mla").with_(d=256, d_cq=256)
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.02, 6, ("w",))
    hidden = ak.normal(6, ("h",), (900, cfg.d))
    streams = ak.latent_streams(ocfg, w, hidden)
    qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [899])
    qn, qr = ak.bf16_round(qn[0]), ak.bf16_round(qr[0])
    want = None
    total = np.zeros((cfg.h, cfg.d_h))
    for k in range(4):
        own = shard_ownership(cfg, 4, k)
        eng = mlra.DecodeEngine(cfg, w, own, batch=1, max_tokens=900)
        rs = _engine_inputs(eng, [streams])[0]
        total[list(own.heads)] = _run(eng, [qn], [qr])[0]
        if want is None:
            want = ak.decode_attention(ocfg, _bf16_weights(w), rs, qn, qr)
    assert ak.max_rel_err(want, total) <= TOL


def test_split_count_invariance_and_batch_independence():
    mlra = _mlra()
    cfg = mlra.trained_config("mlra4").with_(d=256, d_cq=256)
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.02, 8, ("w",))
    lens = [3000, 17, 4097]
    seq_streams, qns, qrs = [], [], []
    for i, n in enumerate(lens):
        hidden = ak.normal(8, ("h", i), (n, cfg.d))
        seq_streams.append(ak.latent_streams(ocfg, w, hidden))
        qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [n - 1])
        qns.append(ak.bf16_round(qn[0]))
        qrs.append(ak.bf16_round(qr[0]))
    outs = []
    for nsplit in (1, 5, 33):
        eng = mlra.DecodeEngine(cfg, w, batch=3, max_tokens=max(lens), nsplit=nsplit)
        _engine_inputs(eng, seq_streams)
        outs.append(_run(eng, qns, qrs))
    for o in outs[1:]:
        assert ak.max_rel_err(outs[0], o) <= TOL_ORDER
    solo = mlra.DecodeEngine(cfg, w, batch=1, max_tokens=max(lens), nsplit=5)
    _engine_inputs(solo, [seq_streams[2]])
    assert ak.max_rel_err(outs[1][2], _run(solo, [qns[2]], [qrs[2]])[0]) <= TOL_ORDER


def test_full_size_tp4_32k_against_oracle_and_permutation():
    """BASELINE configs: TP4 shard of the 2.9B MLRA-4 layer at 32K context (B=2 of the
    B=16 bench batch). Checked against the float64 oracle, and token-permutation invariant
    (attention without a causal mask is order-free: exercises paging/tiling at full size)."""
    mlra = _mlra()
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = mlra.trained_config("mlra4")
    ocfg = _oracle_cfg(cfg)
    n = 32768
    rng = np.random.default_rng(0)
    w = ak.build_weights(ocfg, 0.02, 9, ("w",))
    own = shard_ownership(cfg, 4, 1)
    eng = mlra.DecodeEngine(cfg, w, own, batch=2, max_tokens=n)
    seqs = []
    for i in range(2):
        st = {"latent_b1": rng.standard_normal((n, 128)) * 24 ** 0.5 / 8,
              "rope": rng.standard_normal((n, 64)) * 1.1}
        seqs.append(st)
    qn = [ak.bf16_round(rng.standard_normal((24, 128)) * 2.0) for _ in range(2)]
    qr = [ak.bf16_round(rng.standard_normal((24, 64)) * 0.8) for _ in range(2)]
    rounded = _engine_inputs(eng, seqs)
    got = _run(eng, qn, qr)
    wb = _bf16_weights(w)
    units = ak.shard_units(ocfg, 4, 1)[1]
    for i in range(2):
        cache = ak.Cache(dict(rounded[i]))
        contribs = ak.attend_latent(ocfg, wb, cache, qn[i], qr[i], units)
        want = np.zeros((24, 128))
        for head, vec in contribs:
            want[head] += vec
        want *= 0.5
        assert ak.max_rel_err(want, got[i]) <= TOL
    perm = rng.permutation(n)
    _engine_inputs(eng, [{k: v[perm] for k, v in s.items()} for s in seqs])
    assert ak.max_rel_err(got, _run(eng, qn, qr)) <= TOL_ORDER


def test_first_token_output_is_scaled_branch_value_sum():
    """n = 1 (tests/test_decode.py:68-80): softmax over one token -> alpha * sum_b c_b W^UV_b."""
    mlra = _mlra()
    cfg = mlra.tiny_config()
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.3, 12, ("w",))
    hidden = ak.normal(12, ("h",), (1, cfg.d))
    streams = ak.latent_streams(ocfg, w, hidden)
    qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden, [0])
    eng = mlra.DecodeEngine(cfg, w, batch=1, max_tokens=64)
    rs = _engine_inputs(eng, [streams])[0]
    got = _run(eng, [ak.bf16_round(qn[0])], [ak.bf16_round(qr[0])])[0]
    bs = cfg.block_dim
    wb = _bf16_weights(w)
    expected = sum((rs[f"latent_b{b}"][0] @ wb["w_uv"][b * bs:(b + 1) * bs]).reshape(cfg.h, cfg.d_h) for b in range(4))
    assert ak.max_rel_err(0.5 * expected, got) <= TOL


def test_kimi_64_heads_tp4():
    mlra = _mlra()
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = mlra.table_context()["mlra4"].with_(d=256, d_cq=256)
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.02, 13, ("w",))
    hidden = ak.normal(13, ("h",), (1500, cfg.d))
    streams = ak.latent_streams(ocfg, w, hidden)
    qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [1499])
    qn, qr = ak.bf16_round(qn[0]), ak.bf16_round(qr[0])
    own = shard_ownership(cfg, 4, 2)
    eng = mlra.DecodeEngine(cfg, w, own, batch=1, max_tokens=1500)
    rs = _engine_inputs(eng, [{k: streams[k] for k in ("latent_b2", "rope")}])[0]
    got = _run(eng, [qn], [qr])[0]
    contribs = ak.attend_latent(ocfg, _bf16_weights(w), ak.Cache(dict(rs)), qn, qr, ak.shard_units(ocfg, 4, 2)[1])
    want = np.zeros((64, 128))
    for head, vec in contribs:
        want[head] += vec
    assert ak.max_rel_err(ak.calib_alphas(ocfg)[2] * want, got) <= TOL  # scaling=False here: alpha = 1


@pytest.mark.parametrize("variant", ["mlra", "mla"])
def test_pdl_chained_step_matches_stream_ordered_step(variant, monkeypatch):
    """By default K2 is launched dependent on K1 (programmatic dependent launch: its TMA
    producer streams the cache while K1 drains). Repeated steps and CUDA-graph replays must
    reproduce the plain stream-ordered step (MLRA_NO_PDL=1) exactly -- same kernels, same
    reduction order -- for ragged lengths and both variants."""
    import torch

    mlra = _mlra()
    cfg = mlra.trained_config("mlra4" if variant == "mlra" else "mla").with_(d=256, d_cq=256)
    ocfg = _oracle_cfg(cfg)
    w = ak.build_weights(ocfg, 0.02, 4, ("w",))
    lens = [5, 64, 300, 1000]
    seq_streams, qns, qrs = [], [], []
    for i, n in enumerate(lens):
        hidden = ak.normal(4, ("h", i), (n, cfg.d))
        seq_streams.append(ak.latent_streams(ocfg, w, hidden))
        qn, qr, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [n - 1])
        qns.append(ak.bf16_round(qn[0]))
        qrs.append(ak.bf16_round(qr[0]))
    eng = mlra.DecodeEngine(cfg, w, batch=len(lens), max_tokens=max(lens), page_size=64, nsplit=4)
    rounded = _engine_inputs(eng, seq_streams)
    monkeypatch.setenv("MLRA_NO_PDL", "1")
    base = _run(eng, qns, qrs)
    monkeypatch.delenv("MLRA_NO_PDL", raising=False)
    for _ in range(3):
        got = _run(eng, qns, qrs)
        assert np.array_equal(base, got)
    # graph replay of the PDL-chained step
    qn_t, qr_t = eng.prepare_queries(torch.tensor(np.stack(qns)), torch.tensor(np.stack(qrs)))
    out = eng.decode_attention(qn_t, qr_t)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        eng.decode_attention(qn_t, qr_t, out=out)
    for _ in range(4):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(base, out.double().cpu().numpy())
    wb = _bf16_weights(w)
    for i in range(len(lens)):
        assert ak.max_rel_err(ak.decode_attention(ocfg, wb, rounded[i], qns[i], qrs[i]), got[i]) <= TOL
