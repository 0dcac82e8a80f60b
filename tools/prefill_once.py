"""One prefill_into of n tokens (2.9B MLRA-4 TP1) after a warm-up -- for ncu launch lists / captures."""
import sys, torch
import numpy as np
sys.path.insert(0, ".")
from paper_2603_02188_b200 import decode as dec
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.weights import weight_shapes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
rng = np.random.default_rng(0)
w = {k: rng.standard_normal(s) * 0.02 for k, s in weight_shapes(cfg).items()}
st = dec._state(cfg, w, dev)
h = torch.randn((n, cfg.d), device=dev)
for _ in range(2):
    cache = dec.new_cache(cfg, device=dev, initial_tokens=n)
    dec.prefill_into(cfg, st, cache, h)
torch.cuda.synchronize()
