"""Uniform batch through the device-side split plan vs the uniform split grid (graph replay, two
caches alternated): python tools/plan_uniform.py [tp4|tp1] [B] [ctx]"""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership

lay = sys.argv[1] if len(sys.argv) > 1 else "tp4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
own = shard_ownership(cfg, 4, 0) if lay == "tp4" else None
for mode in ("uniform", "plan"):
    engs = []
    for seed in (21, 22):
        eng, qn, qr = bench.make_engine(cfg, own, B, ctx, seed, dev, ragged=(mode == "plan"))
        engs.append((eng, qn, qr))
    for eng, qn, qr in engs:
        eng.decode_attention(qn, qr)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for i in range(10):
            eng, qn, qr = engs[i % 2]
            eng.decode_attention(qn, qr)
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 50 * 1e3)
    print(f"{lay} B={B} n={ctx} {mode}: {best:.2f} us/step (nsplit {engs[0][0].nsplit})", flush=True)
    del engs, g
    torch.cuda.empty_cache()
