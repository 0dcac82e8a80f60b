"""One warm K4 launch shape (for ncu): B K D from argv."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_02188_b200 import ops
B, K, D = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (16, 3072, 3072)
dev = torch.device("cuda", 0)
attn, gate = torch.randn(B, K, device=dev), torch.randn(B, K, device=dev)
w_o = torch.randn(K, D, device=dev).to(torch.bfloat16)
resid, y = torch.randn(B, D, device=dev), torch.empty(B, D, device=dev)
for _ in range(3):
    ops.outproj(attn, gate, w_o, resid, y)
torch.cuda.synchronize()
print("done")
