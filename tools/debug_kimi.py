import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from decode_check import make_case, reference, rel
from paper_2603_02188_b200 import ops
for (H, ps, lens, nsplit) in [(64, 64, [1500], 1), (64, 128, [1500], 1), (64, 128, [1500], 3), (64, 128, [256], 1), (64, 128, [384], 1), (64,128,[512],1), (48, 128, [1500], 1), (32, 128, [1500], 1)]:
    NB, DLAT, DR, DH = 1, 128, 64, 128
    c = make_case(1, H, DH, NB, DLAT, DR, lens, page_size=ps)
    scale = ops.score_scale((DH + DR) ** -0.5)
    q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
    o_part, lse = ops.decode_partials(q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], ps, NB, 1, 128, nsplit)
    z = ops.combine(o_part, lse, None, 1.0)
    torch.cuda.synchronize()
    zr, _ = reference(c, NB, DLAT, DR, scale, 1.0, q_abs, q_rs)
    bad = [h for h in range(H) if (z[0,0,h]-zr[0,0,h]).abs().max() > 0.05 * zr.abs().max()]
    print(H, ps, lens, nsplit, "rel %.2e" % rel(z, zr), "bad heads", bad[:10], len(bad), flush=True)
