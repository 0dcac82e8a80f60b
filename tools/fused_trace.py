"""Phase timeline of the fused decode step (fused_step.cuh) from the K2 debug trace hook:
per CTA the globaltimer stamps at kernel start, absorb unit done, absorbed queries ready
(grid-wide), partials published, combine done; and the traced CTA's combine sub-phases.

    python tools/fused_trace.py [tp1|tp4|mla] [B] [ctx] [traced cta]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
trace = torch.zeros(16384 + 8 * 160 + 32, dtype=torch.int64, device="cuda")
os.environ["MLRA_DEBUG_TRACE_PTR"] = str(trace.data_ptr())
which = sys.argv[1] if len(sys.argv) > 1 else "tp4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
os.environ["MLRA_DEBUG_TRACE_CTA"] = sys.argv[4] if len(sys.argv) > 4 else "0"
import bench  # noqa: E402
from paper_2603_02188_b200.config import trained_config  # noqa: E402
from paper_2603_02188_b200.tp import shard_ownership  # noqa: E402

cfg = trained_config("mla" if which == "mla" else "mlra4")
own = shard_ownership(cfg, 4, 0) if which in ("tp4", "mla") else None
dev = torch.device("cuda", 0)
eng, qn, qr = bench.make_engine(cfg, own, B, ctx, 1, dev)
for _ in range(3):
    trace.zero_()
    eng.decode_attention(qn, qr)
torch.cuda.synchronize()
t = trace.cpu()
n = eng.nsplit * B
st = t[16384:16384 + 8 * 160].view(160, 8)[:n].double()
t0 = st[:, 0].min()
rel = (st - t0) / 1e3
names = ["start", "absorb unit done", "q~ ready", "partials out", "combine done"]
for k, nm in enumerate(names):
    col = rel[:, k]
    ok = st[:, k] > 0
    if ok.any():
        c = col[ok]
        print(f"{nm:18s} min {c.min():7.2f}  med {c.median():7.2f}  max {c.max():7.2f} us  ({int(ok.sum())} CTAs)")
sub = t[16384 + 8 * 160:16384 + 8 * 160 + 8].double()
lab = {5: "unit start", 0: "seqs ready", 1: "weights", 2: "merged Z", 3: "mma", 4: "unit end"}
print("traced CTA combine:", {lab[k]: round(((sub[k] - t0) / 1e3).item(), 2) for k in (5, 0, 1, 2, 3, 4) if sub[k] > 0})
clk = t[16384 + 8 * 160 + 8:16384 + 8 * 160 + 16].double()
order = [5, 0, 1, 2, 3, 4]
print("traced CTA combine, cycles per phase:", {lab[b]: int(clk[b] - clk[a]) for a, b in zip(order, order[1:]) if clk[a] > 0},
      "-> SM MHz", round(float((clk[4] - clk[5]) / (sub[4] - sub[5]) * 1e3), 0))
