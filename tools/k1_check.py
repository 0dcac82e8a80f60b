import torch, sys
sys.path.insert(0, ".")
from paper_2603_02188_b200 import ops, _lib
dev = torch.device("cuda", 0)
for B, H, DH, NB, DLAT in ((1, 24, 128, 4, 128), (16, 24, 128, 4, 128), (1, 24, 128, 1, 512), (3, 4, 64, 4, 64)):
    qn = torch.randn(B, H, DH, device=dev).to(torch.bfloat16)
    qr = torch.randn(B, H, 64, device=dev).to(torch.bfloat16)
    w = torch.randn(H, DH, NB * DLAT, device=dev).to(torch.bfloat16)
    try:
        qa, qrs = ops.absorb_query(qn, qr, w, NB, DLAT, 0.5)
        ref = torch.einsum("bhk,hkn->bhn", qn.float(), w.float()) * 0.5
        got = qa.float().permute(0, 2, 1, 3).reshape(B, H, NB * DLAT)
        print(B, H, DH, NB, DLAT, "ok", (got - ref).abs().max().item())
    except Exception as e:
        print(B, H, DH, NB, DLAT, "ERR", e)
