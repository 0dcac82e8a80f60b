"""Per-CTA phase timeline of the fused decode step (debug hook MLRA_DEBUG_TRACE_PTR):
start, prologue barrier passed, main loop done, epilogue barrier passed, end."""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
trace = torch.zeros(7 * 256 + 2048 + 8192, dtype=torch.int64, device="cuda")
os.environ["MLRA_DEBUG_TRACE_PTR"] = str(trace.data_ptr())
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.tp import shard_ownership
which = sys.argv[1] if len(sys.argv) > 1 else "tp4"
cfg = trained_config("mla" if which == "mla" else "mlra4")
own = None if which == "tp1" else shard_ownership(cfg, 4, 0)
dev = torch.device("cuda", 0)
eng, qn, qr = bench.make_engine(cfg, own, 16, 32768, 1, dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
for _ in range(3):
    flush.zero_(); trace.zero_(); eng.decode_attention(qn, qr)
torch.cuda.synchronize()
tt = trace.cpu()
cta = tt[7 * 256:7 * 256 + 2048].view(1024, 2)
ph = tt[7 * 256 + 2048:].view(1024, 8)
n = int((cta[:, 1] != 0).sum())
st, en = cta[:n, 0].double(), cta[:n, 1].double()
t0 = st.min()
rel = lambda x: (x.double() - t0) / 1e3
print(f"{which}: CTAs {n}, nsplit {eng.nsplit}")
for name, col in (("start", st), ("absorb_done(w1)", ph[:n, 4]), ("prologue_work", ph[:n, 5]), ("prologue_done", ph[:n, 0]),
                  ("loop_done", ph[:n, 1]), ("epi_barrier", ph[:n, 2]), ("merge_done", ph[:n, 6]), ("end", en)):
    if (col == 0).all():
        print(f"  {name:14s} (not recorded)"); continue
    r = rel(col)
    print(f"  {name:14s} min {r.min().item():7.1f}  med {r.median().item():7.1f}  max {r.max().item():7.1f} us")
seen = ph[:n, 3]
print("  softmax arrivals seen by tid 0 after the final barrier: min", int(seen.min()), "max", int(seen.max()), "(expect 256)")
