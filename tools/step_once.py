"""One warm eager decode step per workload (for ncu launch lists)."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership
dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "tp1"
cfg = trained_config("mlra4")
own = None if which == "tp1" else shard_ownership(cfg, 4, 0)
eng, qn, qr = bench.make_engine(cfg, own, 16, 32768, 1, dev)
for _ in range(3):
    eng.decode_attention(qn, qr)
torch.cuda.synchronize()
print("done")
