"""K4 timing: graph-replayed mlra_outproj (world 1) and the simulated-rank launch, against the
torch path (gate, bf16 cast, cuBLAS GEMM, residual add) for the same shapes."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_02188_b200 import ops

dev = torch.device("cuda", 0)


def gtime(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 10 * 1e3


flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
import os
shapes = [tuple(int(x) for x in a.split(',')) for a in os.environ.get('SHAPES', '16,3072,3072;16,768,3072;1,768,3072;64,3072,3072').split(';')]
for B, K, D in shapes:
    attn = torch.randn(B, K, device=dev)
    gate = torch.randn(B, K, device=dev)
    w_os = [torch.randn(K, D, device=dev).to(torch.bfloat16) for _ in range(8)]  # 8 copies: > L2 when cycled
    resid = torch.randn(B, D, device=dev)
    y = torch.empty(B, D, device=dev)
    it = [0]

    def k4():
        it[0] += 1
        ops.outproj(attn, gate, w_os[it[0] % 8], resid, y)

    def ref():
        it[0] += 1
        a = (attn * torch.sigmoid(gate)).to(torch.bfloat16)
        torch.addmm(resid, a, w_os[it[0] % 8], out=y) if False else y.copy_(resid + (a @ w_os[it[0] % 8]).float())

    t4, tr = gtime(k4), gtime(ref)
    wb = K * D * 2
    print(f"B={B:3d} K={K} D={D}: K4 {t4:6.2f} us ({wb / t4 / 1e3:6.0f} GB/s of W_o)   torch {tr:6.2f} us")
    for world in ((2, 4) if not os.environ.get('NOSIM') else ()):
        if K * world > 3072 * 4:
            continue
        attns = [attn] * world
        gates = [gate] * world
        ys = [torch.empty(B, D, device=dev) for _ in range(world)]
        comms = [torch.zeros(ops.outproj_comm_bytes(B, D, world), dtype=torch.uint8, device=dev) for _ in range(world)]

        def sim():
            ops.outproj_sim(attns, gates, w_os[:world], resid, ys, comms)

        try:
            print(f"      sim world {world}: {gtime(sim):6.2f} us (all ranks on one GPU)")
        except Exception as e:
            print(f"      sim world {world}: {e}")
