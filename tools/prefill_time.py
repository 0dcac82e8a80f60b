"""Prefill timing: prefill_into (projections + K0 + K1 + K6) and K6 alone, 2.9B MLRA-4 TP1, n tokens;
the pseudo-sequence path for comparison. python tools/prefill_time.py [n ...]"""
import sys, torch
import numpy as np
sys.path.insert(0, ".")
from paper_2603_02188_b200 import decode as dec, ops
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.weights import weight_shapes

dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
rng = np.random.default_rng(0)
w = {k: rng.standard_normal(s) * 0.02 for k, s in weight_shapes(cfg).items()}
st = dec._state(cfg, w, dev)

def ev_time(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:]) if len(ts) > 1 else ts[0]

for n in [int(a) for a in sys.argv[1:]] or [1024, 4096, 16384]:
    h = torch.randn((n, cfg.d), device=dev)
    cache = dec.new_cache(cfg, device=dev, initial_tokens=n)
    t_full = ev_time(lambda: dec.prefill_into(cfg, st, cache, h))
    # K6 alone on the filled cache (head-major absorbed queries, as prefill_into builds them)
    kp = st.kproj
    _, _, qn, q_r = kp.project_gemm(h, 0, drq=64)
    w_uk, w_uv = st.lw.packed(cache.layout, dev, st.own)
    sc = ops.score_scale(cfg.tau)  # tau*log2e, as prefill_into applies it (realistic logit range)
    q_abs = (torch.bmm(qn.transpose(0, 1), w_uk).float() * sc).to(torch.bfloat16).view(cfg.h, n, 4, 128)
    q_rs = (q_r.float() * sc).to(torch.bfloat16)
    pc = cache.paged
    t_k6 = ev_time(lambda: ops.prefill_attention(q_abs, q_rs, w_uv, pc.pool, pc.block_table, pc.page_size, 4, 128, 64, 0.5))
    flops = 4 * cfg.h * (n * (n + 1) / 2) * 2 * (128 + 64 + 128) + n * cfg.h * 4 * 128 * 128 * 2 * 2
    t_ps = ev_time(lambda: dec.prefill_into(cfg, st, cache, h, force_pseudo=True), reps=2) if n <= 4096 else float("nan")
    print(f"n={n}: prefill_into {t_full:.3f} ms ({n / t_full * 1e3:.0f} tok/s), K6 {t_k6:.3f} ms "
          f"({flops / t_k6 / 1e9:.0f} TFLOP/s), pseudo-sequence path {t_ps:.3f} ms", flush=True)
