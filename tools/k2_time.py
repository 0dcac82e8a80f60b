"""K2 alone, bench-style: one CUDA graph of 10 launches alternating two caches (B=16, 32K).
usage: python tools/k2_time.py tp1|tp4|mla  (ring override: MLRA_DEBUG_RING=lat,rope,p)"""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.costs import algorithmic_bytes
from paper_2603_02188_b200.tp import shard_ownership
dev = torch.device("cuda", 0)
for which in sys.argv[1:]:
    cfg = trained_config("mla" if which == "mla" else "mlra4")
    own = None if which == "tp1" else shard_ownership(cfg, 4, 0)
    phi = 1 if which == "tp1" else 4
    engs = [bench.make_engine(cfg, own, 16, 32768, s, dev) for s in (1, 2)]
    ms = bench.time_k2_alone(engs, 40)
    nbytes = algorithmic_bytes(cfg, phi, [32768] * 16)
    print(f"{which}: K2 {ms * 1e3:.1f} us  {nbytes / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del engs
    torch.cuda.empty_cache()
