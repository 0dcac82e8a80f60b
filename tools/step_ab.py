import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership
dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
for B, n in ((16, 32768), (1, 131072), (4, 32768)):
    for name, own in (("tp4", shard_ownership(cfg, 4, 0)), ("tp1", None)):
        r = bench.StepRunner(cfg, own, B, n, dev)
        ms = min(bench.time_graph_steps(r, 40, 10, torch.cuda.synchronize) for _ in range(3))
        print(f"{name} B={B} n={n}: step {ms*1e3:.2f} us")
        del r; torch.cuda.empty_cache()
