"""One ragged-batch step per mode (uniform grid, device plan) after warm-up -- for ncu launch lists."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership
dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
own = shard_ownership(cfg, 4, 0)
for ragged in (False, True):
    eng, qn, qr = bench.make_engine(cfg, own, 16, max(bench.RAGGED_LENS), 21, dev, ragged=ragged)
    eng.cache.seqlens.copy_(torch.tensor(bench.RAGGED_LENS, dtype=torch.int32))
    for _ in range(3):
        eng.decode_attention(qn, qr)
    torch.cuda.synchronize()
