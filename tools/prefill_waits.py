"""K6 per-barrier wait cycles of CTA 0 (the longest query tile), n tokens of the 2.9B MLRA-4, on a
dev build of the library: MLRA_NVCC_DEFS=MLRA_PF_WAIT_STATS python -m paper_2603_02188_b200.build
then python tools/prefill_waits.py [n]. Ids as in prefill_kernel.cuh's pf_wait calls."""
import os, sys, torch
import numpy as np
sys.path.insert(0, ".")
from paper_2603_02188_b200 import decode as dec, ops
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.weights import weight_shapes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
rng = np.random.default_rng(0)
w = {k: rng.standard_normal(s) * 0.02 for k, s in weight_shapes(cfg).items()}
st = dec._state(cfg, w, dev)
h = torch.randn((n, cfg.d), device=dev)
cache = dec.new_cache(cfg, device=dev, initial_tokens=n)
dec.prefill_into(cfg, st, cache, h)
torch.cuda.synchronize()
acc = torch.zeros(32, dtype=torch.int64, device=dev)
os.environ["MLRA_DEBUG_PF_WAITS"] = str(acc.data_ptr())
cache = dec.new_cache(cfg, device=dev, initial_tokens=n)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
dec.prefill_into(cfg, st, cache, h)
torch.cuda.synchronize()
names = {1: "prod up_done", 2: "qk q_full", 3: "qk kv_full", 4: "pv p_full", 5: "pv z_full", 6: "pv w_full",
         7: "soft up_done", 8: "soft s_full", 9: "soft pv_done(rescale)", 10: "soft pv_done(P buf)",
         11: "soft pv_done(epi)", 12: "soft up_done(out)", 13: "prod kv_empty", 14: "qk s_empty", 15: "prod kv_empty(W)",
         16: "T branch top", 17: "T s_full wait", 18: "T tmem ld S", 19: "T max+exchange", 20: "T rescale",
         21: "T ex2+pack", 22: "T P-buffer wait", 23: "T P store+arrive", 24: "T branch epilogue", 25: "T OUT store",
         26: "T total (warp 2 lane 0)", 27: "K/V issue -> QK sees it", 28: "count"}
a = acc.cpu().numpy()
print("CTA 0 wait cycles (summed over the threads that waited; softmax ids over 256 threads):")
for i in range(32):
    if a[i]:
        print(f"  {i:2d} {names.get(i, '?'):24s} {a[i]:>14d}")
