"""Per-kernel device times of one decode step (K1, K2, K3) via CUDA-graph replay."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200 import ops
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership

def gtime(fn, iters=50):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            fn()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters / 10 * 1e3

dev = torch.device("cuda", 0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
from paper_2603_02188_b200.config import table_context
tc = table_context()
cases = [("mlra4 tp1", trained_config("mlra4"), None), ("mlra4 tp4 rank", trained_config("mlra4"), shard_ownership(trained_config("mlra4"), 4, 0)),
         ("mla tp4 rank", trained_config("mla"), shard_ownership(trained_config("mla"), 4, 0)),
         ("h64 mlra4 tp4 rank", tc["mlra4"], shard_ownership(tc["mlra4"], 4, 0))]
for name, cfg, own in cases:
    eng, qn, qr = bench.make_engine(cfg, own, B, CTX, 1, dev)
    c = eng.cache
    q_abs, q_rs = ops.absorb_query(qn, qr, eng.w_uk, eng.nb, eng.dlat, eng.scale)
    parts = ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub, eng.dls, eng.nsplit)
    out = ops.combine(*parts, eng.w_uv, eng.alpha)
    scratch = torch.empty((B, len(eng.heads), eng.nb * eng.dlat), dtype=torch.float32, device=dev)
    t1 = gtime(lambda: ops.absorb_query(qn, qr, eng.w_uk, eng.nb, eng.dlat, eng.scale, out=(q_abs, q_rs)))
    t2 = gtime(lambda: ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub, eng.dls, eng.nsplit, out=parts))
    t3 = gtime(lambda: ops.combine(*parts, eng.w_uv, eng.alpha, out=out, scratch=scratch))
    tstep = gtime(lambda: eng.decode_attention(qn, qr))
    print(f"B={B} n={CTX} nsplit={eng.nsplit} {name}: K1 {t1:.1f} us  K2 {t2:.1f} us  K3 {t3:.1f} us  "
          f"step {tstep:.1f} us  (graph replay of 10 launches, one cache: L2-warm)", flush=True)
