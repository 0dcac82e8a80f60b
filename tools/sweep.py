"""Context x batch sweep (BASELINE configs[2] and configs[4]): MLRA-4 TP4 rank and TP1 on one
B200, n in {4K..128K}, B in {1, 4, 16, 64}. Per point: full step (K1+K2+K3, CUDA graph of 10
steps alternating two caches), K2 alone, and the paper's decode scope (K2 + split merge), algorithmic GB/s and fraction of the measured HBM
peak. Writes JSON lines to stdout and a markdown table to gpurun_out/sweep.md."""
import json, os, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.costs import algorithmic_bytes
from paper_2603_02188_b200.tp import shard_ownership

dev = torch.device("cuda", 0)
peak, _ = bench.peaks()
cfg = trained_config("mlra4")
rows = []
ctxs = [4096, 8192, 16384, 32768, 65536, 131072]
batches = [1, 4, 16, 64]
if len(sys.argv) > 1:
    ctxs = [int(x) for x in sys.argv[1].split(",")]
if len(sys.argv) > 2:
    batches = [int(x) for x in sys.argv[2].split(",")]
mla = trained_config("mla")
from paper_2603_02188_b200.config import table_context
tc = table_context()  # the paper's decode benchmark shape: 64 heads, d_h 128, d_h^R 64
layouts = {"tp4_rank": (cfg, shard_ownership(cfg, 4, 0), 4), "tp1": (cfg, None, 1),
           "mla_tp4_rank": (mla, shard_ownership(mla, 4, 0), 4), "mla_tp1": (mla, None, 1),
           "h64_tp4_rank": (tc["mlra4"], shard_ownership(tc["mlra4"], 4, 0), 4),
           "h64_mla_tp4_rank": (tc["mla"], shard_ownership(tc["mla"], 4, 0), 4)}
names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["tp4_rank", "tp1"]
out_md = sys.argv[4] if len(sys.argv) > 4 else "gpurun_out/sweep.md"
for name in names:
    c, own, phi = layouts[name]
    for n in ctxs:
        for B in batches:
            runner = bench.StepRunner(c, own, B, n, dev)
            step_ms = bench.time_graph_steps(runner, 20, 10, torch.cuda.synchronize)
            k2_ms = bench.time_k2_alone(runner.engines, 20)
            ps_ms = bench.time_paper_scope(runner.engines, 20)
            nbytes = algorithmic_bytes(c, phi, [n] * B)
            r = {"layout": name, "ctx": n, "batch": B, "nsplit": runner.engines[0][0].nsplit,
                 "step_us": round(step_ms * 1e3, 2), "step_gbs": round(nbytes / (step_ms * 1e-3) / 1e9, 1),
                 "k2_us": round(k2_ms * 1e3, 2), "k2_gbs": round(nbytes / (k2_ms * 1e-3) / 1e9, 1),
                 "k2_frac": round(nbytes / (k2_ms * 1e-3) / 1e9 / peak, 3),
                 "step_frac": round(nbytes / (step_ms * 1e-3) / 1e9 / peak, 3), "bytes": nbytes,
                 "paper_scope_us": round(ps_ms * 1e3, 2),
                 "paper_scope_frac": round(nbytes / (ps_ms * 1e-3) / 1e9 / peak, 3)}
            print(json.dumps(r), flush=True)
            rows.append(r)
            del runner
            torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
with open(out_md, "w") as f:
    f.write(f"peak (MEASURED_PEAKS hbm_gbs) = {peak} GB/s\n\n")
    f.write("| layout | ctx | B | nsplit | step µs | step GB/s | step frac | K2 µs | K2 GB/s | K2 frac | K2+merge µs | K2+merge frac |\n")
    f.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        f.write(f"| {r['layout']} | {r['ctx']} | {r['batch']} | {r['nsplit']} | {r['step_us']} | {r['step_gbs']} | "
                f"{r['step_frac']} | {r['k2_us']} | {r['k2_gbs']} | {r['k2_frac']} | {r['paper_scope_us']} | "
                f"{r['paper_scope_frac']} |\n")
