import os, sys, torch
sys.path.insert(0, ".")
os.environ["MLRA_DEBUG_FUSE"] = "1"
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership
cfg = trained_config("mlra4")
for B in (16, 8, 12):
    eng, qn, qr = bench.make_engine(cfg, shard_ownership(cfg, 4, 0), B, 4096, 1, torch.device("cuda", 0))
    print("B", B, "nsplit", eng.nsplit, flush=True)
    eng.decode_attention(qn, qr); torch.cuda.synchronize()
