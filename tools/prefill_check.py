"""K6 vs the pseudo-sequence prefill path on one case (debug driver): python tools/prefill_check.py [variant] [n]"""
import faulthandler, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
faulthandler.dump_traceback_later(90, exit=True)
import paper_2603_02188_b200 as mlra
from paper_2603_02188_b200 import decode as dec
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.weights import weight_shapes
from oracle import attnkit_port as ak

variant = sys.argv[1] if len(sys.argv) > 1 else "mlra4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 129
cfg = mlra.tiny_config() if variant == "tiny" else trained_config(variant)
rng = np.random.default_rng(n)
w = {name: rng.standard_normal(shape) * 0.02 for name, shape in weight_shapes(cfg).items()}
dev = torch.device("cuda", 0)
st = dec._state(cfg, w, dev)
h = torch.randn((n, cfg.d), generator=torch.Generator(device=dev).manual_seed(n), device=dev)
outs = []
import os, threading
if os.environ.get("PROGRESS"):
    prog = torch.zeros(8 * 4096, dtype=torch.int32, pin_memory=True)
    os.environ["MLRA_DEBUG_PF_PROGRESS"] = str(prog.data_ptr())
    def dump():
        time.sleep(20)
        a = prog.numpy().reshape(-1, 8)
        nz = [(i, list(a[i])) for i in range(a.shape[0]) if a[i].any()]
        print("progress after 20 s:", len(nz), "CTAs touched", flush=True)
        for i, r in nz[:60]:
            print("  cta", i, r, flush=True)
    threading.Thread(target=dump, daemon=True).start()
if os.environ.get("STEPS"):
    from paper_2603_02188_b200 import ops
    _orig = {k: getattr(ops, k) for k in ("cache_append_latent", "absorb_query", "prefill_attention")}
    def wrap(k):
        def f(*a, **kw):
            print("  launch", k, flush=True)
            r = _orig[k](*a, **kw)
            torch.cuda.synchronize()
            print("  ok", k, flush=True)
            return r
        return f
    for k in _orig:
        setattr(ops, k, wrap(k))
for force in (True, False):
    cache = dec.new_cache(cfg, device=dev, initial_tokens=max(n, 128))
    print("prefill force_pseudo", force, flush=True)
    t0 = time.time()
    o = dec.prefill_into(cfg, st, cache, h, force_pseudo=force)
    torch.cuda.synchronize()
    print("  done", time.time() - t0, flush=True)
    outs.append(o.double().cpu().numpy())
errs = [ak.max_rel_err(outs[0][t], outs[1][t]) for t in range(n)]
print(variant, n, "max_rel_err K6 vs pseudo", max(errs), "at", int(np.argmax(errs)), flush=True)

# float64 reference of the absorbed causal prefill on the SAME bf16 operands (K1's q~ / q_rope,
# the stored cache, the packed W^UV): which path deviates?
from paper_2603_02188_b200 import ops
layout = cache.layout
nb, dlat = dec.kernel_geometry(layout, st.own)
kp = st.kproj
kv_raw, kr_raw, qn, q_r = kp.project_gemm(h, torch.arange(n, dtype=torch.int32, device=dev))
qn, qr = dec._pad_rope(qn, q_r, layout)
qr64 = qr if layout.drp == 64 else torch.nn.functional.pad(qr, (0, 64 - layout.drp))
w_uk, w_uv = st.lw.packed(layout, dev, st.own)
q_abs, q_rs = ops.absorb_query(qn, qr64.contiguous(), w_uk, nb, dlat, ops.score_scale(cfg.tau))
pool = cache.paged.pool.double()
slots = cache.paged.token_slots(0)[:n]
rows = pool[slots]  # [n, W]
C = rows[:, :nb * dlat].reshape(n, nb, dlat)
KR = rows[:, nb * dlat:nb * dlat + layout.dr]
qa = q_abs.double()                    # [n, nb, H, dlat]
qrs = q_rs.double()[..., :layout.dr]   # [n, H, dr]
W = w_uv.double().reshape(cfg.h, nb, dlat, -1)
alpha = 0.5 if cfg.variant == "mlra" else 1.0
ref = torch.zeros((n, cfg.h, W.shape[-1]), dtype=torch.float64, device=dev)
rope_l = torch.einsum("thr,kr->thk", qrs, KR)  # [n, H, n]
mask = torch.triu(torch.ones(n, n, dtype=torch.bool, device=dev), 1)
for b in range(nb):
    lg = torch.einsum("thc,kc->thk", qa[:, b], C[:, b]) + rope_l
    lg = lg.masked_fill(mask[:, None, :], float("-inf"))
    P = torch.softmax(lg * np.log(2.0), dim=-1)
    Z = torch.einsum("thk,kc->thc", P, C[:, b])
    ref += torch.einsum("thc,hcd->thd", Z, W[:, b])
ref = (alpha * ref).cpu().numpy()
for name, o in (("pseudo", outs[0]), ("K6", outs[1])):
    e = [ak.max_rel_err(ref[t], o[t]) for t in range(n)]
    bad = [t for t in range(n) if e[t] > 1e-2]
    print(name, "vs f64 on the same operands: max", max(e), "bad rows", len(bad), bad[:8], bad[-4:], flush=True)

# raw S of one CTA's first key tile (branch 0) vs f64 logits on the same operands
nqt = (n + 127) // 128
cta = 0  # lin 0 -> qt = nqt - 1, head 0
qt, hh = nqt - 1, 0
dbg = torch.zeros(128 * 128, dtype=torch.float32, device=dev)
os.environ["MLRA_DEBUG_PF_S"] = str(dbg.data_ptr())
os.environ["MLRA_DEBUG_PF_CTA"] = str(cta)
ops.prefill_attention(q_abs, q_rs, w_uv, cache.paged.pool, cache.paged.block_table, cache.paged.page_size, nb, dlat,
                      cfg.d_h_rope, alpha)
torch.cuda.synchronize()
del os.environ["MLRA_DEBUG_PF_S"]
S = dbg.view(128, 128).double()
rows_q = torch.arange(qt * 128, qt * 128 + 128, device=dev).clamp(max=n - 1)
want = torch.einsum("tc,kc->tk", qa[rows_q, 0, hh], C[:128, 0]) + torch.einsum("tr,kr->tk", qrs[rows_q, hh], KR[:128])
nk = min(128, n)
d = (S[:, :nk] - want[:, :nk]).abs()
print("S tile0 max abs diff", float(d.max()), "max |S|", float(want.abs().max()), flush=True)
lat_only = torch.einsum("tc,kc->tk", qa[rows_q, 0, hh], C[:128, 0])
print("  vs lat-only logits", float((S[:, :nk] - lat_only[:, :nk]).abs().max()), flush=True)
print("  S[0,:4]", S[0, :4].tolist(), "want", want[0, :4].tolist(), flush=True)
