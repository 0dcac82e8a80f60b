"""Per-round clock64 timeline of CTA (0,0,0) (debug build hook MLRA_DEBUG_TRACE_PTR)."""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from decode_check import make_case
trace = torch.zeros(7 * 256 + 2048, dtype=torch.int64, device="cuda")
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
cta = tt[7 * 256:].view(1024, 2)
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
