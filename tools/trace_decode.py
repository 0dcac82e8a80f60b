"""Per-round clock64 timeline of CTA (0,0,0) (debug build hook MLRA_DEBUG_TRACE_PTR)."""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from decode_check import make_case
trace = torch.zeros(13824 + 2048, dtype=torch.int64, device="cuda")
os.environ["MLRA_DEBUG_TRACE_PTR"] = str(trace.data_ptr())
from paper_2603_02188_b200 import ops
which = sys.argv[1]
NB, DLAT = {"tp4": (1, 128), "tp1": (4, 128), "mla": (1, 512)}[which]
B, H, DH, DR, L = 16, 24, 128, 64, 32768
c = make_case(B, H, DH, NB, DLAT, DR, [L] * B, page_size=128)
sub, dls = ops.latent_geometry(DLAT)
nsplit = ops.default_splits(B, L, NB, sub)
scale = ops.score_scale((DH + DR) ** -0.5)
q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
args = (q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub, dls, nsplit)
o = ops.decode_partials(*args)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_(); ops.decode_partials(*args, out=o)
torch.cuda.synchronize()
tt = trace.cpu()
t = tt[: 7 * 256].view(7, 256)
cta = tt[7 * 256:7 * 256 + 2048].view(1024, 2)
base = t[0, 0].item()
n = int((t[1] != 0).sum())
print("round  tma_issue  data_rdy  qk_issue  S_seen    P_done  pv_issue  mma_done (cycles from first TMA)")
for r in range(min(n, 40)):
    print(f"{r:4d} " + " ".join(f"{(t[e, r].item() - base) if t[e, r] else -1:9d}" for e in (0, 6, 1, 3, 4, 2, 5)))
d = [(t[4, r] - t[4, r - 1]).item() for r in range(5, n)]
print("median round (P_done delta):", sorted(d)[len(d) // 2], "cycles;", "soft busy (P_done - S_seen) median:",
      sorted((t[4, r] - t[3, r]).item() for r in range(5, n))[n // 2 - 3])

n_cta = int((cta[:, 1] != 0).sum())
st = cta[:n_cta, 0].double(); en = cta[:n_cta, 1].double()
t0 = st.min()
dur = (en - st) / 1e3
print(f"CTAs {n_cta}: start spread {(st.max() - t0).item() / 1e3:.1f} us, end max {(en.max() - t0).item() / 1e3:.1f} us, "
      f"dur min/med/max {dur.min().item():.1f}/{dur.median().item():.1f}/{dur.max().item():.1f} us")

import statistics as _st
rr = range(4, n - 4)
def med(xs): return int(_st.median(xs)) if xs else -1
print("median TMA latency (data_rdy - tma_issue):", med([(t[6, r] - t[0, r]).item() for r in rr]),
      "| slot hold (mma_done - data_rdy):", med([(t[5, r] - t[6, r]).item() for r in rr]),
      "| QK->S_seen:", med([(t[3, r] - t[1, r]).item() for r in rr]),
      "| P_done->pv_issue:", med([(t[2, r] - t[4, r]).item() for r in rr]),
      "| period:", med([(t[6, r + 1] - t[6, r]).item() for r in rr]))
sub = tt[12032:12032 + 1024].view(4, 256)
arr = tt[12032 + 1024:12032 + 1280]
print("softmax sub-phases (median cycles): S_seen->S_in_regs", med([(sub[0, r] - t[3, r]).item() for r in rr]),
      "| ->vote", med([(sub[1, r] - sub[0, r]).item() for r in rr]),
      "| ->P slot free", med([(sub[2, r] - sub[1, r]).item() for r in rr]),
      "| ->P stored", med([(sub[3, r] - sub[2, r]).item() for r in rr]),
      "| ->P_done(fence+arrive)", med([(t[4, r] - sub[3, r]).item() for r in rr]))
print("TRUE TMA latency (arrival - issue):", med([(arr[r] - t[0, r]).item() for r in rr]),
      "| arrival -> QK data_rdy seen:", med([(t[6, r] - arr[r]).item() for r in rr]))
e12 = tt[12032 + 5 * 256:12032 + 6 * 256]; e13 = tt[12032 + 6 * 256:12032 + 7 * 256]
print("MMA warp: prev mma_done -> issue_qk entry", med([(e12[r] - t[5, r - 2]).item() for r in rr]),
      "| s_empty wait", med([(e13[r] - e12[r]).item() for r in rr]),
      "| rope+lat wait", med([(t[6, r] - e13[r]).item() for r in rr]))
