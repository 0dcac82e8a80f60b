"""Batch-1 decode steps whose K3 is the merge + head GEMM (64-head and 24-head TP4 ranks, 4K
tokens), for compute-sanitizer: python tools/k3_sanity.py"""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import table_context, trained_config
from paper_2603_02188_b200.tp import shard_ownership

dev = torch.device("cuda", 0)
for name, cfg in (("h64", table_context()["mlra4"]), ("tp4", trained_config("mlra4"))):
    eng, qn, qr = bench.make_engine(cfg, shard_ownership(cfg, 4, 0), 1, 4096, 1, dev)
    out = eng.decode_attention(qn, qr)
    torch.cuda.synchronize()
    eng.check_numeric()
    print(name, "nsplit", eng.nsplit, "out finite", bool(torch.isfinite(out).all()), flush=True)
