"""K5 (peer-memory all-reduce of the TP decode step output) on the GPU: ranks simulated on one
device (one cooperative launch) and two real processes mapping each other's regions through
CUDA IPC. The sum is in ascending rank order, so every rank's result is bit-identical and
equals the float32 left fold of the rank buffers -- exact comparison. Also: graph capture and
replay (the call epoch lives in device memory), ragged sizes, in-place use."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _fold(xs):
    acc = np.zeros_like(xs[0], dtype=np.float32)
    for x in xs:
        acc = (acc + x).astype(np.float32)
    return acc


@pytest.mark.parametrize("world,n", [(2, 49152), (4, 49152), (3, 1000), (8, 4100), (1, 77)])
def test_simulated_ranks_rank_order_sum(world, n):
    from paper_2603_02188_b200 import ops

    rng = np.random.default_rng(world * 1000 + n)
    comms = [torch.zeros(ops.allreduce_comm_bytes(n, world), dtype=torch.uint8, device=DEV) for _ in range(world)]
    for call in range(5):  # both parities, several epochs
        xs = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
        tx = [torch.tensor(x, device=DEV) for x in xs]
        ys = [torch.full((n,), float("nan"), device=DEV) for _ in range(world)]
        ops.allreduce_sim(tx, ys, comms)
        torch.cuda.synchronize()
        want = _fold(xs)
        for r in range(world):
            np.testing.assert_array_equal(ys[r].cpu().numpy(), want)


def test_graph_replay_advances_the_epoch():
    """A captured call replayed many times: fresh epochs every replay, results still exact."""
    from paper_2603_02188_b200 import ops

    world, n = 2, 6000
    comms = [torch.zeros(ops.allreduce_comm_bytes(n, world), dtype=torch.uint8, device=DEV) for _ in range(world)]
    xs = [torch.zeros(n, device=DEV) for _ in range(world)]
    ys = [torch.zeros(n, device=DEV) for _ in range(world)]
    ops.allreduce_sim(xs, ys, comms)  # warm
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ops.allreduce_sim(xs, ys, comms)
    rng = np.random.default_rng(1)
    for _ in range(6):
        vals = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
        for t, v in zip(xs, vals):
            t.copy_(torch.tensor(v))
        g.replay()
        torch.cuda.synchronize()
        for y in ys:
            np.testing.assert_array_equal(y.cpu().numpy(), _fold(vals))


_WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
from paper_2603_02188_b200.collective import PeerAllReduce
rank = int(sys.argv[1])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=rank, world_size=2)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 49152
ar = PeerAllReduce(None, n, dev)
outs = []
for call in range(6):
    x = torch.tensor(np.random.default_rng(10 * call + rank).standard_normal(n).astype(np.float32), device=dev)
    ar(x)  # in place
    outs.append(x)
torch.cuda.synchronize()
np.save(os.path.join(os.environ["OUTDIR"], f"r{rank}.npy"), torch.stack(outs).cpu().numpy())
dist.barrier()
ar.close()
dist.destroy_process_group()
'''


def test_two_processes_over_cuda_ipc(tmp_path):
    import socket

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    env = dict(os.environ, REPO=repo, OUTDIR=str(tmp_path))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), port], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=180)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("IPC worker timed out")
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1)
    for call in range(6):
        xs = [np.random.default_rng(10 * call + r).standard_normal(49152).astype(np.float32) for r in range(2)]
        np.testing.assert_array_equal(r0[call], _fold(xs))


_TP_WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
import paper_2603_02188_b200 as mlra
from paper_2603_02188_b200.collective import PeerAllReduce
from paper_2603_02188_b200.tp import TPDecodeGroup
rank = int(sys.argv[1])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=rank, world_size=2)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for variant in ("mlra4", "mla"):
    cfg = mlra.trained_config(variant)
    B = 4
    red = PeerAllReduce(None, B * cfg.h * cfg.d_h, dev)
    def compute(qn, qr, variant=variant):
        g = torch.Generator(device=dev).manual_seed(rank)
        heads = 24 if variant == "mlra4" else 12
        return torch.randn((B, heads, 128), generator=g, device=dev)
    grp = TPDecodeGroup(cfg, 2, rank, 2, group=None, compute=compute, reducer=red)
    full = torch.empty((B, cfg.h, cfg.d_h), device=dev)
    grp.step(None, None, full)
    torch.cuda.synchronize()
    np.save(os.path.join(os.environ["OUTDIR"], f"{variant}_r{rank}.npy"), full.cpu().numpy())
    dist.barrier()
    red.close()
dist.destroy_process_group()
'''


def test_tp_decode_group_with_peer_reducer(tmp_path):
    """TPDecodeGroup.step with the K5 reducer (two processes, IPC): MLRA-4's all-head partial
    sum and MLA's disjoint head shards both assemble the full output on every rank."""
    import socket

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "tp_worker.py"
    script.write_text(_TP_WORKER)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    env = dict(os.environ, REPO=repo, OUTDIR=str(tmp_path))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), port], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=240)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("TP worker timed out")
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    for variant in ("mlra4", "mla"):
        r0, r1 = np.load(tmp_path / f"{variant}_r0.npy"), np.load(tmp_path / f"{variant}_r1.npy")
        assert np.array_equal(r0, r1)
        parts = []
        for r in range(2):
            g = torch.Generator(device=DEV).manual_seed(r)
            heads = 24 if variant == "mlra4" else 12
            loc = torch.randn((4, heads, 128), generator=g, device=DEV).cpu().numpy()
            full = np.zeros((4, 24, 128), np.float32)
            if variant == "mlra4":
                full[:] = loc
            else:
                full[:, r * 12:(r + 1) * 12] = loc
            parts.append(full)
        np.testing.assert_array_equal(r0, _fold(parts))


_STEP_WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
sys.path.insert(0, os.path.join(os.environ["REPO"], "tests"))
import paper_2603_02188_b200 as mlra
from paper_2603_02188_b200.collective import PeerAllReduce
from paper_2603_02188_b200.tp import shard_ownership
import bench
rank = int(sys.argv[1]); world = int(sys.argv[3])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=rank, world_size=world)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cfg = mlra.trained_config("mlra4")
own = shard_ownership(cfg, world, rank)
outs = {}
for B, ctx in ((16, 2048), (3, 700), (1, 20000)):   # combine4 (fused) and split-K (K5 after) variants
    eng, qn, qr = bench.make_engine(cfg, own, B, ctx, 1000, dev)
    red = PeerAllReduce(None, B * cfg.h * cfg.d_h, dev)
    local = eng.decode_attention(qn, qr).clone()
    fused = [eng.decode_attention_tp(qn, qr, red).clone() for _ in range(3)]
    torch.cuda.synchronize()
    outs[f"local_{B}"] = local.cpu().numpy()
    for i, f in enumerate(fused):
        outs[f"fused_{B}_{i}"] = f.cpu().numpy()
    dist.barrier()
    red.close()
np.savez(os.path.join(os.environ["OUTDIR"], f"step{rank}.npz"), **outs)
dist.destroy_process_group()
'''


@pytest.mark.parametrize("world", [2, 4])
def test_decode_step_with_fused_tp_sum(tmp_path, world):
    """mlra_decode_step_tp in `world` processes on the one GPU (MLRA-4 sharded by latent block,
    every rank holds every head): each rank's fused result equals the float32 rank-order sum of
    the ranks' plain decode outputs, bit-identical across ranks and repeated calls; B = 16 uses
    the fused K3 epilogue, B = 1 long context the split-K K3 followed by K5."""
    import socket

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "step_worker.py"
    script.write_text(_STEP_WORKER)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    env = dict(os.environ, REPO=repo, OUTDIR=str(tmp_path))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), port, str(world)], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for r in range(world)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("step worker timed out")
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    res = [dict(np.load(tmp_path / f"step{r}.npz")) for r in range(world)]
    for B in (16, 3, 1):
        want = _fold([res[r][f"local_{B}"] for r in range(world)])
        for r in range(world):
            for i in range(3):
                np.testing.assert_array_equal(res[r][f"fused_{B}_{i}"], want)
