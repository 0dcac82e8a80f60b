"""Quick GPU numerics check of K1/K2/K3 against a float64 torch restatement (dev tool).

python tools/decode_check.py  -> prints max_rel_err per case, exits 1 on failure.
"""

import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2603_02188_b200 import ops  # noqa: E402


def make_case(B, H, DH, NB, DLAT, DR, lens, page_size=64, seed=0, dev="cuda", contiguous=False):
    g = torch.Generator(device="cpu").manual_seed(seed)
    W = NB * DLAT + DR
    max_len = max(lens)
    max_pages = ops.ceil_div(max_len, page_size) + 1
    num_pages = B * max_pages + 3
    order = torch.arange(num_pages) if contiguous else torch.randperm(num_pages, generator=g)
    perm = order[: B * max_pages].reshape(B, max_pages).to(torch.int32)
    pool = (torch.randn(num_pages * page_size, W, generator=g) * 1.5).to(torch.bfloat16)
    q_nope = torch.randn(B, H, DH, generator=g).to(torch.bfloat16)
    q_rope = torch.randn(B, H, DR, generator=g).to(torch.bfloat16)
    w_uk = (torch.randn(H, DH, NB * DLAT, generator=g) * 0.05).to(torch.bfloat16)
    w_uv = (torch.randn(H, NB * DLAT, DH, generator=g) * 0.05).to(torch.bfloat16)
    seqlens = torch.tensor(lens, dtype=torch.int32)
    return dict(pool=pool.to(dev), bt=perm.to(dev), q_nope=q_nope.to(dev), q_rope=q_rope.to(dev),
                w_uk=w_uk.to(dev), w_uv=w_uv.to(dev), seqlens=seqlens.to(dev), W=W, page_size=page_size)


def reference(c, NB, DLAT, DR, scale, alpha, q_abs=None, q_rs=None):
    pool = c["pool"].double()
    B, H, DH = c["q_nope"].shape
    out = torch.zeros(B, H, DH, dtype=torch.float64, device=pool.device)
    zs = torch.zeros(B, NB, H, DLAT, dtype=torch.float64, device=pool.device)
    ps = c["page_size"]
    for s in range(B):
        n = int(c["seqlens"][s])
        pages = c["bt"][s, : ops.ceil_div(n, ps)].long()
        rows = (pages[:, None] * ps + torch.arange(ps, device=pool.device)[None]).reshape(-1)[:n]
        kv = pool[rows]
        rope = kv[:, NB * DLAT:]
        for b in range(NB):
            lat = kv[:, b * DLAT:(b + 1) * DLAT]
            if q_abs is None:
                qt = torch.einsum("hp,hpc->hc", c["q_nope"][s].double(), c["w_uk"].double()[:, :, b * DLAT:(b + 1) * DLAT]) * scale
                qr = c["q_rope"][s].double() * scale
            else:
                qt = q_abs[s, b].double()
                qr = q_rs[s].double()
            logits = qt @ lat.T + qr @ rope.T  # log2 domain
            p = torch.softmax(logits * math.log(2.0), dim=-1)
            z = p @ lat
            zs[s, b] = z
            out[s] += torch.einsum("hc,hcd->hd", z, c["w_uv"].double()[:, b * DLAT:(b + 1) * DLAT])
    return zs, out * alpha


def rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-30))


def main():
    torch.manual_seed(0)
    cases = [
        # name, B, H, DH, NB, DLAT, DR, lens, nsplit[, page_size]
        ("tiny-tp1-p128", 1, 4, 64, 4, 64, 32, [512], 4, 128),
        ("p-tp4-p128", 3, 24, 128, 1, 128, 64, [1000, 4096, 77], 5, 128),
        ("p-tp1-p256", 3, 24, 128, 4, 128, 64, [1000, 4096, 77], 5, 256),
        ("mla-p128", 2, 24, 128, 1, 512, 64, [2000, 300], 4, 128),
        ("tiny-tp1", 1, 4, 64, 4, 64, 32, [512], 4),
        ("tiny-tp4", 1, 4, 64, 1, 64, 32, [512], 2),
        ("p-tp4", 3, 24, 128, 1, 128, 64, [1000, 4096, 77], 5),
        ("p-tp1", 3, 24, 128, 4, 128, 64, [1000, 4096, 77], 5),
        ("p-tp2", 2, 24, 128, 2, 128, 64, [3000, 129], 3),
        ("mla", 2, 24, 128, 1, 512, 64, [2000, 300], 4),
        ("kimi-tp4", 2, 64, 128, 1, 128, 64, [1500, 64], 3),
        ("mla-tp4-6h", 2, 6, 128, 1, 512, 64, [2500, 65], 3),
    ]
    ok = True
    for name, B, H, DH, NB, DLAT, DR, lens, nsplit, *ps in cases:
        c = make_case(B, H, DH, NB, DLAT, DR, lens, page_size=ps[0] if ps else 64)
        sub, dls = ops.latent_geometry(DLAT)
        scale = ops.score_scale((DH + DR) ** -0.5)
        alpha = 0.5
        q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
        o_part, lse = ops.decode_partials(q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub,
                                          dls, nsplit)
        z = ops.combine(o_part, lse, None, 1.0)
        out = ops.combine(o_part, lse, c["w_uv"], alpha)
        torch.cuda.synchronize()
        zr, _ = reference(c, NB, DLAT, DR, scale, alpha, q_abs, q_rs)
        _, outr = reference(c, NB, DLAT, DR, scale, alpha)
        ez, eo = rel(z, zr), rel(out, outr)
        good = ez < 1e-2 and eo < 2e-2 and torch.isfinite(out).all().item()
        ok &= good
        print(f"{name:12s} z_err={ez:.3e} out_err={eo:.3e} {'OK' if good else 'FAIL'}", flush=True)
    # quick timing of the TP4 / TP1 headline shapes
    for name, NB, DLAT, ps, contig in (("p-tp4 B16 32K", 1, 128, 64, False), ("p-tp4 B16 32K", 1, 128, 128, False),
                                      ("p-tp4 B16 32K", 1, 128, 128, True), ("p-tp1 B16 32K", 4, 128, 128, False),
                                      ("mla B16 32K", 1, 512, 128, False)):
        B, H, DH, DR, L = 16, 24, 128, 64, 32768
        name = f"{name} page={ps}{' contiguous' if contig else ''}"
        c = make_case(B, H, DH, NB, DLAT, DR, [L] * B, page_size=ps, contiguous=contig)
        sub, dls = ops.latent_geometry(DLAT)
        nsplit = ops.default_splits(B, L, NB, sub)
        scale = ops.score_scale((DH + DR) ** -0.5)
        q_abs, q_rs = ops.absorb_query(c["q_nope"], c["q_rope"], c["w_uk"], NB, DLAT, scale)
        args = (q_abs, q_rs, c["pool"], c["bt"], c["seqlens"], c["page_size"], NB, sub, dls, nsplit)
        o = ops.decode_partials(*args)
        for _ in range(3):
            ops.decode_partials(*args, out=o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(10):
            flush.zero_()
            e0.record()
            ops.decode_partials(*args, out=o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = sorted(ts)[len(ts) // 2]
        nbytes = B * L * (NB * DLAT + DR) * 2
        print(f"{name}: nsplit={nsplit} {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s", flush=True)
    print("ALL OK" if ok else "SOME FAILED")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
