"""One eager K1 / K2 / K3 per workload (for ncu duration lists of the small kernels)."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200 import ops
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership
dev = torch.device("cuda", 0)
for name, cfg, own in [("tp1", trained_config("mlra4"), None),
                       ("tp4", trained_config("mlra4"), shard_ownership(trained_config("mlra4"), 4, 0))]:
    eng, qn, qr = bench.make_engine(cfg, own, 16, 32768, 1, dev)
    c = eng.cache
    for _ in range(3):
        q_abs, q_rs = ops.absorb_query(qn, qr, eng.w_uk, eng.nb, eng.dlat, eng.scale)
        parts = ops.decode_partials(q_abs, q_rs, c.pool, c.block_table, c.seqlens, c.page_size, eng.nb, eng.sub, eng.dls, eng.nsplit)
        out = ops.combine(*parts, eng.w_uv, eng.alpha)
    torch.cuda.synchronize()
    print(name, "done", flush=True)
