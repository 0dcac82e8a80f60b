import sys, os, math, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from decode_check import make_case, reference, rel
from paper_2603_02188_b200 import ops
print("threshold", os.environ.get("MLRA_DEBUG_RESCALE_THRESHOLD"))
for (NB, H, DLAT, lens, nsplit) in [(1,24,512,[128],1),(1,6,512,[128],1),(1,24,512,[192],1),(1,24,512,[640],1)]:
    DH, DR = 128, 64
    c = make_case(1, H, DH, NB, DLAT, DR, lens)
    sub, dls = ops.latent_geometry(DLAT)
    scale = ops.score_scale((DH + DR) ** -0.5)
    q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
    outs = []
    for rep in range(4):
        o_part, lse = ops.decode_partials(q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], 64, NB, sub, dls, nsplit)
        outs.append(ops.combine(o_part, lse, None, 1.0))
    torch.cuda.synchronize()
    z = outs[0]
    det = all(torch.equal(outs[0], o) for o in outs[1:])
    zr, _ = reference(c, NB, DLAT, DR, scale, 1.0, q_abs, q_rs)
    err_cols = [(z[0,:,:,i*64:(i+1)*64]-zr[0,:,:,i*64:(i+1)*64]).abs().max().item() for i in range(DLAT//64)]
    print(NB, H, DLAT, lens, nsplit, "rel %.2e" % rel(z, zr), "deterministic", det, "cols", ["%.2f"%e for e in err_cols], flush=True)
