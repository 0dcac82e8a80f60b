"""Per-CTA pipeline summary of K2 (debug trace hook MLRA_DEBUG_TRACE_PTR / MLRA_DEBUG_TRACE_CTA):
for several CTAs, the median TMA latency, slot hold, softmax time and round period."""
import os, sys, statistics as st, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from decode_check import make_case
trace = torch.zeros(13824 + 2048, dtype=torch.int64, device="cuda")
os.environ["MLRA_DEBUG_TRACE_PTR"] = str(trace.data_ptr())
from paper_2603_02188_b200 import ops
which = sys.argv[1]
NB, DLAT = {"tp4": (1, 128), "tp1": (4, 128), "mla": (1, 512), "h64": (1, 128)}[which]
B, H, DH, DR = 16, 64 if which == "h64" else 24, 128, 64
B = int(os.environ.get("TRACE_B", B)); L = int(os.environ.get("TRACE_L", 32768))
c = make_case(B, H, DH, NB, DLAT, DR, [L] * B, page_size=128)
c2 = make_case(B, H, DH, NB, DLAT, DR, [L] * B, page_size=128, seed=1)  # the bench alternates two caches
sub, dls = ops.latent_geometry(DLAT)
nsplit = ops.default_splits(B, L, NB, sub)
scale = ops.score_scale((DH + DR) ** -0.5)
q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
args = (q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub, dls, nsplit)
o = ops.decode_partials(*args)
args2 = (q_abs, q_rs, c2["pool"], c2["bt"], c2["seqlens"], c2["page_size"], NB, sub, dls, nsplit)
o2 = ops.decode_partials(*args2)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
def med(xs): return int(st.median(xs)) if xs else -1
ctas = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 8, 40, 77, 100, 135, 143]
print("prologue (cycles from CTA start): producer start, page ids in, first TMA")
for cta in ctas[:1]:
    pass
print("cta  dur_us  rounds period tma_lat  hold  soft  Pdone->PV  QK->S | start->TMA0 TMA0->data0 data0->Pdone0 lastPV->softdone ->ofinal ->stored ->end (cycles)")
for cta in ctas:
    os.environ["MLRA_DEBUG_TRACE_CTA"] = str(cta)
    for _ in range(3):
        trace.zero_(); ops.decode_partials(*args2, out=o2); ops.decode_partials(*args, out=o)
    torch.cuda.synchronize()
    tt = trace.cpu()
    t = tt[: 7 * 256].view(7, 256)
    ce = tt[7 * 256:7 * 256 + 2048].view(1024, 2)
    n = int((t[1] != 0).sum())
    arr = t[6]
    ep = tt[7 * 256 + 2048 + 8 * cta: 7 * 256 + 2048 + 8 * cta + 8]
    rr = range(3, n - 2)
    dur = (ce[cta, 1] - ce[cta, 0]).item() / 1e3
    print(f"{cta:3d} {dur:7.1f} {n:6d} {med([(t[6, r + 1] - t[6, r]).item() for r in rr]):6d} "
          f"{med([(arr[r] - t[0, r]).item() for r in rr]):7d} "
          f"{med([(t[5, r] - t[6, r]).item() for r in rr]):5d} {med([(t[4, r] - t[3, r]).item() for r in rr]):5d} "
          f"{med([(t[2, r] - t[4, r]).item() for r in rr]):10d} {med([(t[3, r] - t[1, r]).item() for r in rr]):6d} | "
          f"{(t[0, 0] - tt[13824 + 2 * cta]).item():10d} {(arr[0] - t[0, 0]).item():11d} {(t[4, 0] - arr[0]).item():13d} "
          f"{(ep[3] - t[5, n - 1]).item():16d} {(ep[4] - ep[3]).item():7d} {(ep[5] - ep[4]).item():7d} {(tt[13824 + 2 * cta + 1] - ep[5]).item():5d}"
          f" | prod-start {(tt[13056] - tt[13824 + 2 * cta]).item()} pages-in {(tt[13057] - tt[13824 + 2 * cta]).item()}"
          f" bar7 {(tt[13058] - tt[13824 + 2 * cta]).item()} rope-tma {(tt[13059] - tt[13824 + 2 * cta]).item()}")
n_cta = int((ce[:, 1] != 0).sum())
s0 = ce[:n_cta, 0].double(); e0 = ce[:n_cta, 1].double()
d = ((e0 - s0) / 1e3)
ck = tt[13824:13824 + 2 * n_cta].view(n_cta, 2).double()
mhz = (ck[:, 1] - ck[:, 0]) / (e0 - s0) * 1e3
print(f"SM clock over CTA lifetimes: min/med/max {mhz.min().item():.0f}/{mhz.median().item():.0f}/{mhz.max().item():.0f} MHz")
print(f"all {n_cta} CTAs: dur min/med/max {d.min().item():.1f}/{d.median().item():.1f}/{d.max().item():.1f} us; "
      f"end spread {(e0.max() - e0.min()).item() / 1e3:.1f} us")
srt = sorted(range(n_cta), key=lambda i: d[i].item())
print("fastest:", [(i, round(d[i].item(), 1)) for i in srt[:6]], "slowest:", [(i, round(d[i].item(), 1)) for i in srt[-6:]])
