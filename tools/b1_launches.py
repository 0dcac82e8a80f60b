"""One eager decode step per small-batch workload (B = 1; 24-head TP4 rank at 4K / 128K, the
64-head TP4 rank at 128K), for an ncu launch list of K1 / K2 / K3 durations:
ncu --metrics gpu__time_duration.sum --csv --log-file L python tools/b1_launches.py [case,...]"""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import table_context, trained_config
from paper_2603_02188_b200.tp import shard_ownership

dev = torch.device("cuda", 0)
tc = table_context()
cases = [("tp4_4k", trained_config("mlra4"), 4096), ("tp4_128k", trained_config("mlra4"), 131072),
         ("h64_128k", tc["mlra4"], 131072)]
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for name, cfg, ctx in cases:
    if only is not None and name not in only:
        continue
    eng, qn, qr = bench.make_engine(cfg, shard_ownership(cfg, 4, 0), 1, ctx, 1, dev)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(name)
    for _ in range(3):
        eng.decode_attention(qn, qr)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(name, "nsplit", eng.nsplit, flush=True)
