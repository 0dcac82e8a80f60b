"""Run one decode_partials config repeatedly (for ncu). usage: prof_decode.py tp4|tp1|mla [iters]"""
import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from decode_check import make_case
from paper_2603_02188_b200 import ops
which = sys.argv[1]; iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
NB, DLAT = {"tp4": (1, 128), "tp1": (4, 128), "mla": (1, 512)}[which]
B, H, DH, DR, L = 16, 24, 128, 64, 32768
c = make_case(B, H, DH, NB, DLAT, DR, [L] * B, page_size=128)
sub, dls = ops.latent_geometry(DLAT)
nsplit = int(sys.argv[3]) if len(sys.argv) > 3 else ops.default_splits(B, L, NB, sub)
scale = ops.score_scale((DH + DR) ** -0.5)
q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
args = (q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub, dls, nsplit)
o = ops.decode_partials(*args)
for _ in range(iters):
    ops.decode_partials(*args, out=o)
torch.cuda.synchronize()
print("done", which, nsplit)
