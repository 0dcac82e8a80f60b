"""Step time vs split count at small batches (graph of 10 alternating steps over two caches,
like bench.StepRunner): python tools/split_sweep.py tp4|tp1|h64|mla|h64mla B ctx nsplit,nsplit,..."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200 import ops
from paper_2603_02188_b200.config import trained_config, table_context
from paper_2603_02188_b200.tp import shard_ownership

lay, B, ctx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
cfg = {"h64": lambda: table_context()["mlra4"], "mla": lambda: trained_config("mla"),
       "h64mla": lambda: table_context()["mla"]}.get(lay, lambda: trained_config("mlra4"))()
own = shard_ownership(cfg, 4, 0) if lay in ("tp4", "h64", "mla", "h64mla") else None
engs = [bench.make_engine(cfg, own, B, ctx, 1000 + i, dev) for i in range(2)]
default = engs[0][0].nsplit
vals = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [default]
for v in vals:
    if v > default:
        continue
    for eng, _, _ in engs:
        eng.nsplit = v
        eng.workspace = ops.DecodeWorkspace(B, len(eng.heads), eng.nb, eng.dlat, eng.layout.drp, v, eng.device)
    for eng, qn, qr in engs:
        eng.decode_attention(qn, qr)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(10):
            eng, qn, qr = engs[i % 2]
            eng.decode_attention(qn, qr)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 100 * 1e3)
    print(f"{lay} B={B} n={ctx} nsplit={v} (default {default}): step {best:.2f} us", flush=True)
