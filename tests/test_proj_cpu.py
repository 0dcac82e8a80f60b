"""Host-side packing of the K-1 projection kernels (no GPU): the slab-packed weight layout the
kernels stream (include/mlra_b200.h) and the pre-multiplied W^UQ.W^UK_b query weight, checked
against the reference's own arithmetic (attnkit/latent.py:129-139, decode.py:155-167)."""

import numpy as np
import torch

from oracle import attnkit_port as ak
from paper_2603_02188_b200 import ops
from paper_2603_02188_b200.config import AttnConfig
from paper_2603_02188_b200.decode import _write_plan, full_ownership, kernel_geometry, local_weights, row_layout
from paper_2603_02188_b200.projections import KernelProjector
from paper_2603_02188_b200.tp import shard_ownership


def test_slab_pack_layout():
    """[K, N] -> [ceil(N/64)][round_up(K, 64)][64]: element [s][k][c] = W[k][64 s + c], zero
    outside W (a slab's columns are one contiguous run per K row)."""
    rng = np.random.default_rng(0)
    for K, N in ((100, 70), (64, 64), (3072, 1600), (33, 8)):
        w = torch.as_tensor(rng.standard_normal((K, N)), dtype=torch.float32).to(torch.bfloat16)
        p = ops.slab_pack(w)
        assert tuple(p.shape) == ops.slab_shape(K, N) == (-(-N // 64), -(-K // 64) * 64, 64)
        full = torch.zeros((p.shape[1], p.shape[0] * 64), dtype=torch.bfloat16)
        full[:K, :N] = w
        for s in range(p.shape[0]):
            assert torch.equal(p[s], full[:, 64 * s:64 * s + 64])


def _cfg():
    return AttnConfig("mlra", branches=4, h=8, d=64, d_h=16, d_h_rope=8, d_c=64, d_cq=32)


def test_preabsorbed_query_weight_is_wuq_times_wuk():
    """For a one-block owner the query weight's first columns are W^UQ_h . W^UK_(b),(h)^T in
    (branch, head, latent) order: c_q . W^Q equals absorb_query(q_nope) of the reference."""
    cfg = _cfg()
    ocfg = ak.cfg_from(cfg)
    w = ak.build_weights(ocfg, 0.1, 3, ("proj-cpu",))
    own = shard_ownership(cfg, 4, 2)
    layout = row_layout(cfg, own)
    nb, dlat = kernel_geometry(layout, own)
    uk, _ = local_weights(cfg, w, own).packed_host(layout, own)
    kp = KernelProjector(cfg, w, "cpu", own.heads, _write_plan(cfg, own)[0], uk_pack=uk, nb=nb, dlat=dlat,
                         drp=layout.drp, absorbed=True, score_scale=1.0)
    assert kp.absorbed and kp.q_shape == (nb, len(own.heads), dlat)
    c_q = np.random.default_rng(1).standard_normal((3, cfg.d_cq))
    got = c_q @ kp.w_query.float().numpy()[:, :kp.nq].astype(np.float64)
    q_nope = (c_q @ w["w_uq"]).reshape(3, cfg.h, cfg.d_h)
    block = 2  # shard_ownership(mlra4, 4, k) owns latent block k
    bs = cfg.d_c // 4
    w_uk_b = w["w_uk"][block * bs:(block + 1) * bs]  # (latent, h*d_h)
    for i in range(3):
        want = ak.absorb_query(q_nope[i], w_uk_b)  # [h, latent]
        assert ak.max_rel_err(want, got[i].reshape(nb, cfg.h, dlat)[0, :, :bs]) < 2e-2  # bf16 weight


def test_down_weight_concatenation_and_kv_slices():
    """w_down = [W^DQ | W^DKV | W^KR]; kv_slice picks the owner's raw latent columns."""
    cfg = _cfg()
    w = ak.build_weights(ak.cfg_from(cfg), 0.1, 4, ("proj-cpu",))
    names = _write_plan(cfg, full_ownership(cfg))[0]
    kp = KernelProjector(cfg, w, "cpu", range(cfg.h), names, absorbed=False)
    want = np.concatenate([w["w_dq"], *[w[n] for n in names], w["w_kr"]], axis=1)
    assert kp.w_down.shape == want.shape
    np.testing.assert_allclose(kp.w_down.float().numpy(), ak.bf16_round(want), rtol=0, atol=0)
    assert (kp.n_q, kp.n_kv, kp.n_kr) == (cfg.d_cq, cfg.d_c, cfg.d_h_rope)
    kv = torch.arange(2 * kp.n_kv, dtype=torch.float32).reshape(2, kp.n_kv)
    assert torch.equal(kp.kv_slice(kv, names), kv)
