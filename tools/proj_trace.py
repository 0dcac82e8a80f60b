"""Per-CTA phase stamps of one K-1 launch (globaltimer ns, relative to the earliest CTA start):
0 start, 1 after griddepcontrol.wait, 2 X staged, 3 first W box, 4 GEMM done, 5 cluster barrier."""
import os, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership

dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
eng, hid = bench.make_layer_engine(cfg, shard_ownership(cfg, 4, 0), 16, 1024, 5, dev)
kp = eng.kernel_projector(None)
kp.down(hid); kp.query(16, eng.cache.seqlens); torch.cuda.synchronize()
tr = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
os.environ["MLRA_DEBUG_PROJ_TRACE"] = str(tr.data_ptr())
for name, fn in (("down", lambda: kp.down(hid)), ("query", lambda: kp.query(16, eng.cache.seqlens))):
    for rep in range(3):
        tr.zero_(); torch.cuda.synchronize()
        fn(); torch.cuda.synchronize()
    t = tr.view(-1, 8).cpu()
    n = int((t[:, 0] > 0).sum())
    t = t[:n].double()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"{name}: {n} CTAs")
    for k, lab in enumerate(["start", "waited", "x staged", "first box", "gemm done", "cluster"]):
        col = rel[:, k]
        ok = t[:, k] > 0
        col = col[ok]
        if len(col):
            print(f"  {lab:10s} min {col.min():6.2f} med {col.median():6.2f} max {col.max():6.2f} us")
