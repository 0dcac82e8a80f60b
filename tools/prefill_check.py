"""K6 vs the pseudo-sequence prefill path on one case (debug driver): python tools/prefill_check.py [variant] [n]"""
import faulthandler, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
faulthandler.dump_traceback_later(900, exit=True)
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
    prog = torch.zeros(16 * 4096, dtype=torch.int32, pin_memory=True)
    os.environ["MLRA_DEBUG_PF_PROGRESS"] = str(prog.data_ptr())
    def dump():
        time.sleep(20)
        a = prog.numpy().reshape(-1, 16)
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

for t0 in range(0, n, 128):
    e = max(errs[t0:t0 + 128])
    hs = [max(ak.max_rel_err(outs[0][t, hh], outs[1][t, hh]) for t in range(t0, min(n, t0 + 128))) for hh in range(outs[0].shape[1])]
    print(f"  tile {t0 // 128}: {e:.3e} per head {[f'{x:.1e}' for x in hs[:8]]}", flush=True)
