"""Step and K2-alone times (graph replay, two caches alternated) for one layout under the current
environment: python tools/step_env.py [tp4|tp1|h64] [B] [ctx]. Run once per MLRA_* dev setting."""
import os, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership

lay = sys.argv[1] if len(sys.argv) > 1 else "tp4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
dev = torch.device("cuda", 0)
from paper_2603_02188_b200.config import table_context
cfg = table_context()["mlra4"] if lay == "h64" else trained_config("mlra4")
own = shard_ownership(cfg, 4, 0) if lay in ("tp4", "h64") else None
r = bench.StepRunner(cfg, own, B, ctx, dev)
step = min(bench.time_graph_steps(r, 40, 10, torch.cuda.synchronize) for _ in range(5)) * 1e3
k2 = min(bench.time_k2_alone(r.engines, 20) for _ in range(3)) * 1e3
env = {k: v for k, v in os.environ.items() if k.startswith("MLRA_")}
print(f"{lay} B={B} n={ctx} env={env}: step {step:.2f} us  K2 {k2:.2f} us", flush=True)
