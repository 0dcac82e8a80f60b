"""K-1 (pre-attention projections, csrc/proj_kernel.cuh) against the reference's
latent_projections (attnkit/latent.py:129-159): golden q_nope / q_rope rows from the real
reference, and the oracle port on the same bf16 weights (float64 math) for the raw
down-projections, the rotary queries at large positions and the pre-absorbed query q~."""

import numpy as np
import pytest
import torch

import paper_2603_02188_b200 as mlra
from oracle import attnkit_port as ak
from paper_2603_02188_b200 import ops
from paper_2603_02188_b200.decode import _write_plan, full_ownership, kernel_geometry, local_weights, row_layout
from paper_2603_02188_b200.projections import KernelProjector
from paper_2603_02188_b200.tp import shard_ownership
import golden_util as gu

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
LATENT_CASES = ("tiny_mlra4", "refdims_mlra4", "refdims_mla", "p_mlra4", "p_mla", "p_mlra2", "p_gla2",
                "refdims_mlra2", "refdims_gla2")


def _projector(cfg, w, absorbed=False, own=None):
    own = own or full_ownership(cfg)
    names = _write_plan(cfg, full_ownership(cfg))[0]
    if not absorbed:
        return KernelProjector(cfg, w, DEV, own.heads, names, absorbed=False)
    layout = row_layout(cfg, own)
    lw = local_weights(cfg, w, own)
    nb, dlat = kernel_geometry(layout, own)
    uk, _ = lw.packed(layout, DEV, own)
    return KernelProjector(cfg, w, DEV, own.heads, names, uk_pack=uk.float().cpu().numpy(), nb=nb, dlat=dlat,
                           drp=layout.drp, absorbed=True, score_scale=ops.score_scale(cfg.tau))


def _bf16_weights(w):
    return {k: ak.bf16_round(np.asarray(v)) for k, v in w.items()}


@pytest.mark.parametrize("case", LATENT_CASES)
def test_queries_match_reference_golden(case):
    """The last token's q_nope / q_rope from K-1 vs the real reference's (golden, float64).
    Error budget: bf16 weights and bf16 outputs (~2^-9 relative each)."""
    meta, g = gu.load(case)
    cfg, w, hidden = gu.regen(meta)
    n = meta["n"]
    mcfg = mlra.AttnConfig(**meta["cfg"])
    kp = _projector(mcfg, w)
    _, _, qn, qr = kp.project(torch.as_tensor(hidden[n - 1:], dtype=torch.float32, device=DEV),
                              torch.tensor([n - 1], dtype=torch.int32, device=DEV))
    qn = qn[0].double().cpu().numpy()
    qr = qr[0, :, :cfg.d_h_rope].double().cpu().numpy()
    e1, e2 = ak.max_rel_err(g["q_nope"], qn), ak.max_rel_err(g["q_rope"], qr)
    assert e1 < 1e-2 and e2 < 1e-2, (case, e1, e2)


@pytest.mark.parametrize("case", ("p_mlra4", "p_mla", "p_gla2", "refdims_mlra2"))
def test_raw_projections_exact_on_bf16_weights(case):
    """kv_raw / kr_raw (fp32 outputs) for 20 rows (two launches of <= 16) vs float64 on the
    same bf16 weights: the hi/lo activation split keeps them within ~1e-5."""
    meta, _ = gu.load(case)
    cfg, w, hidden = gu.regen(meta)
    mcfg = mlra.AttnConfig(**meta["cfg"])
    kp = _projector(mcfg, w)
    rows = hidden[:20] if hidden.shape[0] >= 20 else np.concatenate([hidden] * (20 // hidden.shape[0] + 1))[:20]
    kv, kr, _, _ = kp.project(torch.as_tensor(rows, dtype=torch.float32, device=DEV),
                              torch.arange(20, dtype=torch.int32, device=DEV))
    wb = _bf16_weights(w)
    x = rows.astype(np.float32).astype(np.float64)
    want_kv = np.concatenate([x @ wb[nm] for nm in kp.kv_names], axis=1)
    want_kr = x @ wb["w_kr"]
    assert ak.max_rel_err(want_kv, kv.double().cpu().numpy()) < 2e-5
    assert ak.max_rel_err(want_kr, kr.double().cpu().numpy()) < 2e-5


def test_rope_queries_at_large_positions():
    """q_rope at positions up to 131071 (fp64 angle reduction in the epilogue) and 16 rows with
    distinct positions, against the oracle on the same bf16 weights."""
    meta, _ = gu.load("p_mlra4")
    cfg, w, hidden = gu.regen(meta)
    mcfg = mlra.AttnConfig(**meta["cfg"])
    kp = _projector(mcfg, w)
    pos = [0, 1, 7, 63, 64, 1000, 4095, 4096, 32767, 32768, 65535, 65536, 100000, 131000, 131070, 131071]
    rows = hidden[:16]
    _, _, qn, qr = kp.project(torch.as_tensor(rows, dtype=torch.float32, device=DEV),
                              torch.tensor(pos, dtype=torch.int32, device=DEV))
    wb = _bf16_weights(w)
    q_nope, q_rope, _, _ = ak.latent_projections(cfg, wb, rows.astype(np.float32).astype(np.float64), pos)
    for i in range(16):
        assert ak.max_rel_err(q_nope[i], qn[i].double().cpu().numpy()) < 6e-3, i
        assert ak.max_rel_err(q_rope[i], qr[i, :, :cfg.d_h_rope].double().cpu().numpy()) < 6e-3, i


@pytest.mark.parametrize("variant", ("mlra4", "mlra2"))
def test_preabsorbed_query_matches_absorb(variant):
    """TP4 rank (one latent block): the pre-multiplied W^UQ.W^UK_b projection writes K2's q~
    = tau*log2e * q_nope . W^UK_b^T directly (K1 skipped) -- vs the oracle's absorb_query."""
    case = {"mlra4": "p_mlra4", "mlra2": "p_mlra2"}[variant]
    meta, _ = gu.load(case)
    cfg, w, hidden = gu.regen(meta)
    mcfg = mlra.AttnConfig(**meta["cfg"])
    own = shard_ownership(mcfg, 4, 1)
    kp = _projector(mcfg, w, absorbed=True, own=own)
    assert kp.absorbed and kp.q_shape[0] == 1
    n = meta["n"]
    _, _, qa, qr = kp.project(torch.as_tensor(hidden[n - 4:], dtype=torch.float32, device=DEV),
                              torch.arange(n - 4, n, dtype=torch.int32, device=DEV))
    q_nope, q_rope, _, _ = ak.latent_projections(cfg, w, hidden[n - 4:], list(range(n - 4, n)))
    s = float(ops.score_scale(mcfg.tau))
    layout = row_layout(mcfg, own)
    uk, _ = local_weights(mcfg, w, own).packed(layout, DEV, own)
    ukf = uk.double().cpu().numpy()  # [H, d_h, DLAT] (zero where a unit does not serve a head)
    for i in range(4):
        want = s * np.einsum("hp,hpc->hc", q_nope[i][list(own.heads)], ukf)
        got = qa[i, 0].double().cpu().numpy()
        assert ak.max_rel_err(want, got) < 1.5e-2, i
        want_r = s * q_rope[i][list(own.heads)]
        assert ak.max_rel_err(want_r, qr[i, :, :cfg.d_h_rope].double().cpu().numpy()) < 1e-2, i
