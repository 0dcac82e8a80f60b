"""Multi-process TP plumbing on CPU (gloo, world size 2): each rank owns the units
`shard_ownership` assigns it, computes its share (here with the CPU oracle in place of the
GPU kernels -- the injectable `compute`), and one all_reduce(SUM) reproduces the
single-device result, for MLRA-4 (branch sum) and MLA (disjoint heads = concat)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import attnkit_port as ak
from paper_2603_02188_b200.config import AttnConfig
from paper_2603_02188_b200.tp import TPDecodeGroup, group_ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(variant, batch=2, n=40):
    if variant == "mlra":
        cfg = AttnConfig("mlra", branches=4, h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16, scaling=True)
    else:
        cfg = AttnConfig("mla", h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16, scaling=True)
    ocfg = ak.cfg_from(cfg)
    w = ak.build_weights(ocfg, 0.3, 11, ("w",))
    seqs = []
    for s in range(batch):
        hidden = ak.normal(11, ("h", s), (n + s, cfg.d))
        streams = ak.latent_streams(ocfg, w, hidden)
        q_nope, q_rope, _, _ = ak.latent_projections(ocfg, w, hidden[-1:], [n + s - 1])
        seqs.append((streams, q_nope[0], q_rope[0]))
    return cfg, ocfg, w, seqs


def _worker(rank, world, port, variant, tp, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, ocfg, w, seqs = _problem(variant)
        groups = [dist.new_group(r) for r in group_ranks(world, tp)]
        grp = TPDecodeGroup(cfg, tp, rank, world, group=groups[rank // tp])
        alpha = ak.calib_alphas(ocfg)[2] if cfg.variant == "mlra" else 1.0
        units = ak.shard_units(ocfg, tp, grp.tp_rank)[1]

        def compute(q_nope, q_rope):  # this rank's share for its batch slice (oracle stand-in)
            outs = []
            for (streams, qn, qr) in seqs_local:
                contribs = ak.attend_latent(ocfg, w, ak.Cache(dict(streams)), qn, qr, units)
                local = np.zeros((len(grp.own.heads), cfg.d_h))
                pos = {h: i for i, h in enumerate(grp.own.heads)}
                for head, vec in contribs:
                    local[pos[head]] += vec
                outs.append(alpha * local)
            return torch.tensor(np.stack(outs))

        sl = grp.batch_slice(len(seqs))
        seqs_local = seqs[sl]
        grp.compute = compute
        full = torch.zeros((len(seqs_local), cfg.h, cfg.d_h), dtype=torch.float64)
        grp.step(None, None, full)
        out_q.put((rank, sl.start, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant,tp", [("mlra", 2), ("mla", 2), ("mlra", 1)])
def test_tp_group_allreduce_matches_single_device(variant, tp):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, variant, tp, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, ocfg, w, seqs = _problem(variant)
    for rank, start, full in results:
        for i in range(full.shape[0]):
            streams, qn, qr = seqs[start + i]
            ref = ak.decode_attention(ocfg, w, streams, qn, qr)
            assert ak.max_rel_err(ref, full[i]) <= 1e-10, (rank, i)
    if tp == 2:  # both ranks of the single TP group hold the same reduced result
        assert np.allclose(results[0][2], results[1][2])


def test_group_layout():
    assert group_ranks(8, 4) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert group_ranks(4, 4) == [[0, 1, 2, 3]]
    assert group_ranks(2, 1) == [[0], [1]]


def _reducer_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench

        group = dist.new_group([0, 1])
        red, kind = bench.make_reducer("nccl", group, 8, torch.device("cpu"))
        res = [(red is None, kind)]
        # no GPU here: K5's region allocation fails, the bench falls back to the collective
        red, kind = bench.make_reducer("peer", group, 8, torch.device("cpu"))
        res.append((red is None, kind))
        # the TP group's reducer hook replaces its all_reduce
        calls = []

        def reducer(t):
            calls.append(t.numel())
            dist.all_reduce(t, group=group)
            return t

        cfg = AttnConfig("mla", h=4, d=32, d_h=8, d_h_rope=4, d_c=32, d_cq=16, scaling=True)
        grp = TPDecodeGroup(cfg, 2, rank, world, group=group, reducer=reducer,
                            compute=lambda qn, qr: torch.full((1, 2, 8), float(rank + 1), dtype=torch.float64))
        full = torch.zeros((1, 4, 8), dtype=torch.float64)
        grp.step(None, None, full)
        res.append((calls, full[0, :, 0].tolist()))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_bench_reducer_fallback_and_tp_group_hook():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reducer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        (none_nccl, kind_nccl), (none_peer, kind_peer), (calls, col) = results[rank]
        assert none_nccl and kind_nccl == "nccl all_reduce"
        assert none_peer and kind_peer.startswith("nccl all_reduce (K5 unavailable")
        assert calls == [32]
        assert col == [1.0, 1.0, 2.0, 2.0]  # MLA: rank r owns heads 2r, 2r+1
