"""K-1 timing: proj_down and proj_query alone (CUDA graphs of 10, two weight sets alternated so
the weights come from HBM), at the 2.9B shape, B = 16, TP4 rank (pre-absorbed) -- usage:
python tools/proj_time.py [KS]"""
import os, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership

dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
engs = [bench.make_layer_engine(cfg, shard_ownership(cfg, 4, 0), 16, 1024, 5 + i, dev) for i in range(2)]
kps = [e.kernel_projector(None) for e, _ in engs]

def gtime(fns, reps=50):
    for f in fns: f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for i in range(10): fns[i % len(fns)]()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 10 * 1e3

down = [lambda i=i: kps[i].down(engs[i][1]) for i in range(2)]
query = [lambda i=i: kps[i].query(16, engs[i][0].cache.seqlens) for i in range(2)]
both = [lambda i=i: (kps[i].down(engs[i][1]), kps[i].query(16, engs[i][0].cache.seqlens)) for i in range(2)]
kp = kps[0]
bd, bq = kp.w_down.numel() * 2, kp.w_query.numel() * 2
td, tq, tb = gtime(down), gtime(query), gtime(both)
print(f"KS env={os.environ.get('MLRA_DEBUG_PROJ_KS')}: down {td:.2f} us ({bd/td/1e3:.0f} GB/s, {bd/1e6:.1f} MB)  "
      f"query {tq:.2f} us ({bq/tq/1e3:.0f} GB/s, {bq/1e6:.1f} MB)  both {tb:.2f} us")
