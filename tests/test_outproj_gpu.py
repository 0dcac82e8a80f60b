"""K4 (output side) on the GPU against the oracle: gate + W_o + residual
(attnkit/zoo.py:125-152) and the fused one-shot all-reduce, with the ranks simulated on one
device (mlra_outproj_sim: the same kernel, one cooperative launch) and, in the last test, as
two processes mapping each other's regions through CUDA IPC.

Tolerance: the gated operand and W_o are bf16 on the tensor cores (fp32 accumulation). Against
an oracle fed the same bf16-rounded operands the error is fp32 summation order plus the odd
operand whose bf16 rounding flips with the fast sigmoid (gate 1e-4 of the projection's scale;
1e-5 without a gate); against the exact float64 reference output it is bounded by
the bf16 rounding of the operands (2e-2 of the projection's scale)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import attnkit_port as ak

from golden_util import load, regen_outproj

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _t(a, dtype=torch.float32):
    return torch.tensor(np.asarray(a), dtype=torch.float32).to(DEV, dtype).contiguous()


def _oracle_bf16(hidden, parts, w_o, w_g, d_h, resid=True):
    """tp_attention_block_output with the kernel's operand rounding (gated A and W_o in bf16)."""
    acc = np.zeros((hidden.shape[0], w_o.shape[1]))
    for heads, out_r in parts:
        cols = np.concatenate([np.arange(i * d_h, (i + 1) * d_h) for i in heads])
        g = out_r * ak.sigmoid(hidden @ w_g[:, cols]) if w_g is not None else out_r
        acc = acc + ak.bf16_round(g.astype(np.float32)) @ ak.bf16_round(w_o[cols])
    return (hidden if resid else 0.0) + acc


def _check(got, want, base, tol):
    scale = max(np.abs(want - base).max(), 1e-30)
    err = np.abs(got - want).max() / scale
    assert err <= tol, f"rel err {err:.3e} > {tol}"


@pytest.mark.parametrize("gated", [True, False])
def test_single_rank_matches_reference_golden(gated):
    from paper_2603_02188_b200 import ops

    meta, arr = load("outproj_p")
    cfg, w, hidden, flat = regen_outproj(meta)
    gate_pre = _t(hidden @ w["w_g"]) if gated else None
    y = torch.empty((hidden.shape[0], cfg.d), dtype=torch.float32, device=DEV)
    ops.outproj(_t(flat), gate_pre, _t(w["w_o"], torch.bfloat16), _t(hidden), y)
    got = y.double().cpu().numpy()
    want = arr["y_gated" if gated else "y_plain"]
    _check(got, _oracle_bf16(hidden, [(range(cfg.h), flat)], w["w_o"], w["w_g"] if gated else None, cfg.d_h), hidden,
           1e-4)
    _check(got, want, hidden, 2e-2)


@pytest.mark.parametrize("world,by", [(2, "heads"), (4, "heads"), (4, "branches"), (3, "heads")])
def test_simulated_ranks_sum_in_rank_order(world, by):
    """world ranks on one device: every rank's y is bit-identical and equals the device-order sum."""
    from paper_2603_02188_b200 import ops

    meta, arr = load("outproj_p")
    cfg, w, hidden0, _ = regen_outproj(meta)
    rng = np.random.default_rng(world)
    B, h, d_h = 16, cfg.h, cfg.d_h
    if by == "heads" and h % world:
        h = 24  # 24 heads split 3 ways
    hidden = rng.standard_normal((B, cfg.d))
    if by == "heads":
        per = h // world
        parts = [(list(range(r * per, (r + 1) * per)), rng.standard_normal((B, per * d_h)) * 0.5) for r in range(world)]
    else:
        parts = [(list(range(h)), rng.standard_normal((B, h * d_h)) * 0.5) for _ in range(world)]
    w_o, w_g = w["w_o"], w["w_g"]
    cols = [np.concatenate([np.arange(i * d_h, (i + 1) * d_h) for i in hs]) for hs, _ in parts]
    attns = [_t(o) for _, o in parts]
    gates = [_t(hidden @ w_g[:, c]) for c in cols]
    w_os = [_t(w_o[c], torch.bfloat16) for c in cols]
    ys = [torch.full((B, cfg.d), float("nan"), device=DEV) for _ in range(world)]
    comms = [torch.zeros(ops.outproj_comm_bytes(B, cfg.d, world), dtype=torch.uint8, device=DEV) for _ in range(world)]
    ops.outproj_sim(attns, gates, w_os, _t(hidden), ys, comms)
    torch.cuda.synchronize()
    for r in range(1, world):
        assert torch.equal(ys[r], ys[0]), f"rank {r} differs from rank 0"
    _check(ys[0].double().cpu().numpy(), _oracle_bf16(hidden, parts, w_o, w_g, d_h), hidden, 1e-4)
    _check(ys[0].double().cpu().numpy(), ak.tp_attention_block_output(hidden, parts, w_o, w_g, d_h), hidden, 2e-2)


def test_epochs_alternate_buffers_across_many_calls():
    """Eight back-to-back calls (both parities, inputs changing every call, no host sync in
    between) on 2 simulated ranks; also B > 16 (row groups), a K tail and a D tail."""
    from paper_2603_02188_b200 import ops

    rng = np.random.default_rng(0)
    world, B, K, D = 2, 40, 72, 200
    w_o = [rng.standard_normal((K, D)) * 0.1 for _ in range(world)]
    comms = [torch.zeros(ops.outproj_comm_bytes(B, D, world), dtype=torch.uint8, device=DEV) for _ in range(world)]
    ys_all, wants = [], []
    for call in range(8):
        hidden = rng.standard_normal((B, D))
        attn = [rng.standard_normal((B, K)) for _ in range(world)]
        gpre = [rng.standard_normal((B, K)) for _ in range(world)]
        ys = [torch.empty((B, D), device=DEV) for _ in range(world)]
        ops.outproj_sim([_t(a) for a in attn], [_t(g) for g in gpre], [_t(x, torch.bfloat16) for x in w_o], _t(hidden),
                        ys, comms)
        ys_all.append(ys)
        want = hidden.copy()
        for r in range(world):
            want += ak.bf16_round((attn[r] * ak.sigmoid(gpre[r])).astype(np.float32)) @ ak.bf16_round(w_o[r])
        wants.append((hidden, want))
    torch.cuda.synchronize()
    for ys, (hidden, want) in zip(ys_all, wants):
        assert torch.equal(ys[0], ys[1])
        _check(ys[0].double().cpu().numpy(), want, hidden, 1e-4)


def test_output_projection_module_single_rank():
    """OutputProjection (the host API) for a TP4 head shard of MLA and for MLRA-4's full-head
    branch partial: y equals the oracle's block output of what the rank holds."""
    import paper_2603_02188_b200 as mlra
    from paper_2603_02188_b200.outproj import OutputProjection

    meta, _ = load("outproj_p")
    cfg_o, w, _, _ = regen_outproj(meta)
    rng = np.random.default_rng(3)
    for variant, heads in (("mla", list(range(6, 12))), ("mlra4", list(range(24)))):
        cfg = mlra.trained_config(variant).with_(gated=True)
        B = 5
        hidden = rng.standard_normal((B, cfg.d))
        attn = rng.standard_normal((B, len(heads), cfg.d_h)) * 0.3
        op = OutputProjection(cfg, w, heads, batch=B, device=DEV)
        y = op(_t(attn), _t(hidden)).double().cpu().numpy()
        parts = [(heads, attn.reshape(B, -1))]
        _check(y, _oracle_bf16(hidden, parts, w["w_o"], w["w_g"], cfg.d_h), hidden, 1e-4)
        y0 = op(_t(attn), _t(hidden), residual=False).double().cpu().numpy()
        _check(y0, _oracle_bf16(hidden, parts, w["w_o"], w["w_g"], cfg.d_h, resid=False), 0.0, 1e-4)


_IPC_WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
from paper_2603_02188_b200 import ops
from paper_2603_02188_b200.outproj import TpComm
rank = int(sys.argv[1]); world = 2
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=rank, world_size=world)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
B, K, D = 8, 128, 256
comm = TpComm(None, B, D, dev)
ys = []
for call in range(4):
    rng = np.random.default_rng(100 * call + rank)
    attn = torch.tensor(rng.standard_normal((B, K)), dtype=torch.float32, device=dev)
    w_o = torch.tensor(rng.standard_normal((K, D)) * 0.1, dtype=torch.float32, device=dev).to(torch.bfloat16)
    resid = torch.tensor(np.random.default_rng(7 + call).standard_normal((B, D)), dtype=torch.float32, device=dev)
    y = torch.empty((B, D), device=dev)
    ops.outproj(attn, None, w_o, resid, y, rank, world, comm.ptrs)
    ys.append(y)
torch.cuda.synchronize()
np.save(os.path.join(os.environ["OUTDIR"], f"y{rank}.npy"), torch.stack(ys).cpu().numpy())
dist.barrier()
comm.close()
dist.destroy_process_group()
'''


def test_two_processes_over_cuda_ipc(tmp_path):
    """The real multi-process path (TpComm: comm_alloc + IPC handles over a gloo group, peer
    regions opened with cudaIpcOpenMemHandle) with both processes on the one GPU."""
    import socket

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "worker.py"
    script.write_text(_IPC_WORKER)
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
    y0, y1 = np.load(tmp_path / "y0.npy"), np.load(tmp_path / "y1.npy")
    assert np.array_equal(y0, y1)
    B, K, D = 8, 128, 256
    for call in range(4):
        want = np.random.default_rng(7 + call).standard_normal((B, D)).astype(np.float32).astype(np.float64)
        for r in range(2):
            rng = np.random.default_rng(100 * call + r)
            attn = rng.standard_normal((B, K))
            w_o = rng.standard_normal((K, D)) * 0.1
            want = want + ak.bf16_round(attn.astype(np.float32)) @ ak.bf16_round(w_o.astype(np.float32))
        _check(y0[call], want, 0.0, 1e-5)


def test_graph_replay_of_the_all_reduce_path():
    """K4 with 2 simulated ranks captured once and replayed with new inputs: the device-side
    epoch advances every replay (both receive-buffer parities), results stay exact."""
    from paper_2603_02188_b200 import ops

    rng = np.random.default_rng(9)
    world, B, K, D = 2, 8, 128, 256
    w_o = [_t(rng.standard_normal((K, D)) * 0.1, torch.bfloat16) for _ in range(world)]
    attn = [torch.zeros((B, K), device=DEV) for _ in range(world)]
    resid = torch.zeros((B, D), device=DEV)
    ys = [torch.empty((B, D), device=DEV) for _ in range(world)]
    comms = [torch.zeros(ops.outproj_comm_bytes(B, D, world), dtype=torch.uint8, device=DEV) for _ in range(world)]
    ops.outproj_sim(attn, None, w_o, resid, ys, comms)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ops.outproj_sim(attn, None, w_o, resid, ys, comms)
    for _ in range(5):
        a = [rng.standard_normal((B, K)) for _ in range(world)]
        hid = rng.standard_normal((B, D))
        for t, v in zip(attn, a):
            t.copy_(_t(v))
        resid.copy_(_t(hid))
        g.replay()
        torch.cuda.synchronize()
        want = hid + sum(ak.bf16_round(a[r].astype(np.float32)) @ ak.bf16_round(w_o[r].float().cpu().numpy())
                         for r in range(world))
        assert torch.equal(ys[0], ys[1])
        _check(ys[0].double().cpu().numpy(), want, hid, 1e-5)
