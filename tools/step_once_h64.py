"""One warm eager decode step at the paper's 64-head shape (TP4 rank, B=1, 1M context), for ncu."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import table_context
from paper_2603_02188_b200.tp import shard_ownership
dev = torch.device("cuda", 0)
cfg = table_context()["mlra4"]
eng, qn, qr = bench.make_engine(cfg, shard_ownership(cfg, 4, 0), 1, 1 << 20, 1, dev)
for _ in range(3):
    eng.decode_attention(qn, qr)
torch.cuda.synchronize()
print("done")
