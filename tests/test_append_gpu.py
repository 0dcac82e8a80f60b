"""GPU parity of the fused write side (K0: rmsnorm * alpha_kv + block split + RoPE + paged
append, mlra_cache_append_latent) against the oracle's latent_projections
(attnkit/latent.py:129-159), including RoPE at 128K-scale positions, a TP4 shard's single
block, and MLA's undivided latent. Rows are stored in bf16: gate = bf16 rounding of the
oracle's float64 row (relative 2^-8 of the row's max)."""

import numpy as np
import pytest
import torch

from oracle import attnkit_port as ak

pytestmark = pytest.mark.gpu


def _check(variant, own_blocks, positions):
    import paper_2603_02188_b200 as mlra
    from paper_2603_02188_b200.cache import PagedCache
    from paper_2603_02188_b200.decode import _write_plan, full_ownership, row_layout
    from paper_2603_02188_b200.tp import shard_ownership

    cfg = mlra.trained_config("mla" if variant == "mla" else "mlra4").with_(d=512)
    ocfg = ak.cfg_from(cfg)
    w = ak.build_weights(ocfg, 0.02, 3, ("k0",))
    own = full_ownership(cfg) if own_blocks is None else shard_ownership(cfg, 4, own_blocks)
    lay = row_layout(cfg, own)
    B = len(positions)
    hidden = ak.normal(3, ("k0-h",), (B, cfg.d))
    dev = torch.device("cuda", 0)
    cache = PagedCache(lay, B, 256, 64, dev)
    h = torch.tensor(hidden, dtype=torch.float32, device=dev)
    _, branches, block0, nblocks, norm_groups = _write_plan(cfg, own)
    alpha_kv = ak.calib_alphas(ocfg)[1]
    kv_raw = torch.tensor(hidden @ w["w_dkv"], dtype=torch.float32, device=dev)
    kr_raw = torch.tensor(hidden @ w["w_kr"], dtype=torch.float32, device=dev)
    cache.append_latent(kv_raw, kr_raw, positions, branches=branches, block0=block0, nblocks=nblocks,
                        alpha_kv=alpha_kv, norm_groups=norm_groups)
    torch.cuda.synchronize()
    del h
    for s, pos in enumerate(positions):
        _, _, k_rope, lats = ak.latent_projections(ocfg, w, hidden[s:s + 1], [pos])
        row = cache.pool[cache.token_slots(s)][0]
        for name in list(lay.units) + ["rope"]:
            want = (k_rope if name == "rope" else lats[name])[0]
            got = lay.extract(name, row[None]).double().cpu().numpy()[0]
            err = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30)
            assert err <= 2 ** -7, f"{variant} seq {s} pos {pos} stream {name}: rel err {err:.3e}"
        pad = row[lay.width - lay.drp + lay.dr:]
        assert float(pad.abs().max() if pad.numel() else 0.0) == 0.0


@pytest.mark.parametrize("variant,blocks", [("mlra", None), ("mlra", 2), ("mla", None)])
def test_fused_append_matches_oracle(variant, blocks):
    _check(variant, blocks, [0, 1, 17, 4095, 65537, 131071])


def test_fused_append_through_drop_in_step_tracks_packed_rows():
    """absorbed_decode_step appends through the fused K0: the stored rows equal the oracle's
    latent streams (bf16) token by token."""
    import paper_2603_02188_b200 as mlra

    cfg = mlra.tiny_config()
    ocfg = ak.cfg_from(cfg)
    w = ak.build_weights(ocfg, 0.3, 5, ("k0s",))
    hidden = ak.normal(5, ("k0s-h",), (20, cfg.d))
    cache = mlra.new_cache(cfg, pos_offset=1000)
    for t in range(20):
        mlra.absorbed_decode_step(cfg, w, cache, hidden[t])
    streams = ak.latent_streams(ocfg, w, hidden, pos_offset=1000)
    for name, want in streams.items():
        got = cache.peek(name)
        assert np.max(np.abs(got - want)) <= 2 ** -7 * np.max(np.abs(want)), name


def test_plain_append_advance_flag():
    """mlra_cache_append: the row lands at positions[s]; advance=1 bumps positions (the
    reference append grows the cache, cache.py:44-57), advance=0 leaves them alone."""
    from paper_2603_02188_b200 import ops

    dev = torch.device("cuda", 0)
    B, W, ps, maxp = 5, 320, 64, 4
    pool = torch.zeros((B * maxp * ps, W), dtype=torch.bfloat16, device=dev)
    bt = torch.randperm(B * maxp, generator=torch.Generator().manual_seed(1)).to(torch.int32).reshape(B, maxp).to(dev)
    pos0 = torch.tensor([0, 63, 64, 200, 253], dtype=torch.int32)
    pos = pos0.clone().to(dev)
    for step, adv in enumerate([False, True, True]):
        rows = (torch.arange(B * W, dtype=torch.float32).reshape(B, W) % 251 + 100 * step).to(torch.bfloat16).to(dev)
        before = pos.cpu()
        ops.cache_append(rows, bt, pos, pool, ps, advance=adv)
        torch.cuda.synchronize()
        assert torch.equal(pos.cpu(), before + (1 if adv else 0))
        for s in range(B):
            p = int(before[s])
            slot = int(bt[s, p // ps]) * ps + p % ps
            assert torch.equal(pool[slot], rows[s])
    assert torch.equal(pos.cpu(), pos0 + 2)


@pytest.mark.parametrize("graphs", [False, True])
def test_micro_batch_loop_matches_in_order_steps(graphs):
    """host_loop.MicroBatchLoop (one H2D / D2H per step on side streams, K0 advance, two
    micro-batches interleaved; with graphs, K1..K3 replayed from a per-micro-batch CUDA graph
    after the first step) gives exactly the outputs and cache of the plain in-order calls."""
    import paper_2603_02188_b200 as mlra
    from paper_2603_02188_b200 import DecodeEngine
    from paper_2603_02188_b200.host_loop import MicroBatchLoop

    cfg = mlra.trained_config("mlra4")
    rng = np.random.default_rng(5)
    w = {"w_uk": rng.standard_normal((cfg.d_c, cfg.h * cfg.d_h)) * 0.02,
         "w_uv": rng.standard_normal((cfg.d_c, cfg.h * cfg.d_h)) * 0.02}
    dev = torch.device("cuda", 0)
    B, n0, steps = 3, 300, 4

    def engines():
        out = []
        for k in range(2):
            e = DecodeEngine(cfg, w, batch=B, max_tokens=n0 + 64, page_size=64, device=dev)
            g = torch.Generator(device=dev).manual_seed(10 + k)
            e.cache.pool.copy_((torch.randn(e.cache.pool.shape, generator=g, device=dev) * 0.3).to(torch.bfloat16))
            e.cache.seqlens.fill_(n0 - k)
            e.cache._host_lens = [n0 - k] * B
            out.append(e)
        return out

    ea, eb = engines(), engines()
    loop = MicroBatchLoop(ea, graphs=graphs)
    g = torch.Generator().manual_seed(3)
    host = [[[torch.randn(t.shape, generator=g).to(torch.bfloat16) for t in loop.host_inputs(k)]
             for k in range(2)] for _ in range(steps)]
    got, want = [], []
    for i in range(steps):
        for k in range(2):
            for dst, src in zip(loop.host_inputs(k), host[i][k]):
                dst.copy_(src)
            loop.submit(k)
        for k in range(2):
            got.append(loop.wait(k).clone())
    for i in range(steps):
        for k in range(2):
            rows, qn, qr = (t.to(dev) for t in host[i][k])
            eb[k].cache.append(rows)
            want.append(eb[k].decode_attention(qn, qr).cpu().clone())
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        assert torch.equal(a, b)
    for a, b in zip(ea, eb):
        assert torch.equal(a.cache.seqlens, b.cache.seqlens)
        assert a.cache.lengths() == b.cache.lengths() == [n0 + steps - (a is ea[1])] * B
        assert torch.equal(a.cache.pool, b.cache.pool)
