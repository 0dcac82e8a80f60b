"""Per-round timeline of one K2 CTA (debug trace hook): distribution of round periods and the
longest stalls, in the bench-like setting (two caches, back to back)."""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from decode_check import make_case
trace = torch.zeros(13824 + 2048, dtype=torch.int64, device="cuda")
os.environ["MLRA_DEBUG_TRACE_PTR"] = str(trace.data_ptr())
os.environ["MLRA_DEBUG_TRACE_CTA"] = sys.argv[2] if len(sys.argv) > 2 else "0"
from paper_2603_02188_b200 import ops
which = sys.argv[1]
NB, DLAT = {"tp4": (1, 128), "tp1": (4, 128), "mla": (1, 512)}[which]
B, H, DH, DR, L = 16, 24, 128, 64, 32768
cs = [make_case(B, H, DH, NB, DLAT, DR, [L] * B, page_size=128, seed=s) for s in (0, 1)]
sub, dls = ops.latent_geometry(DLAT)
nsplit = ops.default_splits(B, L, NB, sub)
scale = ops.score_scale((DH + DR) ** -0.5)
q_abs, q_rs = ops.absorb_query(cs[0]["q_nope"], cs[0]["q_rope"], cs[0]["w_uk"], NB, DLAT, scale)
outs = [ops.decode_partials(q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub, dls, nsplit) for c in cs]
for _ in range(3):
    trace.zero_()
    for i in (1, 0):
        c = cs[i]
        ops.decode_partials(q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub, dls, nsplit, out=outs[i])
torch.cuda.synchronize()
tt = trace.cpu()
t = tt[: 7 * 256].view(7, 256)
n = int((t[1] != 0).sum())
P = [(t[4, r] - t[4, r - 1]).item() for r in range(1, n)]
Ps = sorted(P)
print(f"rounds {n}; P_done period: min {Ps[0]} p10 {Ps[len(Ps)//10]} med {Ps[len(Ps)//2]} p90 {Ps[9*len(Ps)//10]} max {Ps[-1]}; "
      f"mean {sum(P)/len(P):.0f}")
print("round:period for the 12 longest:", sorted(((p, r + 1) for r, p in enumerate(P)), reverse=True)[:12])
# waits: data_rdy (6) vs qk entry (12-> index 12032+5*256) and TMA issue (0)
e13 = tt[12032 + 6 * 256:12032 + 7 * 256]
print("per round r (first 24): period, TMA issue->data seen, s_empty seen->data seen, P_done->PV issue")
for r in range(1, min(n, 25)):
    print(f"  r{r:3d} {P[r-1]:6d} {(t[6, r] - t[0, r]).item():7d} {(t[6, r] - e13[r]).item():7d} {(t[2, r] - t[4, r]).item():6d}")
