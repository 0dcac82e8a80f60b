"""Summarise ncu captures into profiles/ (ncu_summary.json)."""
import csv, json, os, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (v[i], units[i]) for i, k in enumerate(h)}

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]

def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)

summary = json.load(open("profiles/ncu_summary.json")) if os.path.exists("profiles/ncu_summary.json") else {}
for name, rep, algo, kname in [
        ("mlra4_tp1_b16_n32768", "gpurun_out/k2_tp1.ncu-rep", 603979776, "mlra_decode_kernel (K2)"),
        ("mlra4_tp4_b16_n32768", "gpurun_out/k2_tp4.ncu-rep", 201326592, "mlra_decode_kernel (K2)"),
        ("outproj_b16_k3072_d3072", "gpurun_out/k4.ncu-rep", 3072 * 3072 * 2, "outproj_allreduce_kernel (K4, world 1)"),
        # K-1: the weight-streaming projection GEMMs (algorithmic bytes = the down weight of one launch)
        ("proj_down_b16_k3072_n1600", "gpurun_out/proj.ncu-rep", 3072 * 1600 * 2, "proj_gemm_kernel (K-1 down)"),
        # K6: causal prefill, n = 4096 (bytes are not its bound: the tensor pipe is; traffic recorded)
        ("prefill_mlra4_tp1_n4096", "gpurun_out/k6.ncu-rep", 4096 * (1152 + 24 * 512 * 2 + 24 * 64 * 2 + 24 * 128 * 4),
         "prefill_attention_kernel (K6; tensor-bound: bytes = cache + q~ + q_rope + out)"),
        # batch-1 K3 at the paper's 64-head shape (TP4 rank, 128K, 148 splits): the merge reads the
        # split partials + lse and writes Z; the head GEMM reads W^UV (64 x 128 x 128 bf16) + Z
        ("merge_h64_b1_n131072", "gpurun_out/k3m.ncu-rep", 148 * 64 * 128 * 4 + 148 * 64 * 4 + 64 * 128 * 4,
         "merge_splits_kernel<16> (K3 merge, 32 columns x 16 split groups)"),
        ("headgemm_h64_b1", "gpurun_out/k3g.ncu-rep", 64 * 128 * 128 * 2 + 2 * 64 * 128 * 4,
         "head_gemm_kernel (K3 up-projection, PDL)"),
        # the paper's 64-head shape at batch 1, 1M tokens (TP4 rank: one 128-wide latent + rope)
        ("mlra4_h64_tp4_b1_n1048576", "gpurun_out/k2_h64.ncu-rep", 1048576 * 192 * 2, "mlra_decode_kernel (K2, 64 heads)"),
        # K3 at TP1, B = 16, 32K: split partials + lse + W^UV (4 branches x 24 heads) + output
        ("combine4_tp1_b16", "gpurun_out/k3_tp1.ncu-rep",
         16 * 9 * 4 * 24 * 128 * 4 + 16 * 9 * 4 * 24 * 4 + 4 * 24 * 128 * 128 * 2 + 16 * 24 * 128 * 4,
         "combine4_kernel<4> (K3 merge + W^UV + cluster branch sum)")]:
    if not os.path.exists(rep):
        continue
    r = raw(rep)
    dur_unit = r["gpu__time_duration.sum"][1]
    dur_us = float(r["gpu__time_duration.sum"][0].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[dur_unit]
    rd = to_bytes(*r["dram__bytes_read.sum"])
    wr = to_bytes(*r["dram__bytes_write.sum"])
    summary[name] = {
        "kernel": kname, "duration_us_ncu": dur_us, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr, "algorithmic_bytes": algo, "traffic_over_algorithmic": round((rd + wr) / algo, 4),
        "metrics": {k: " ".join(r[k]) for k in WANT if k in r},
        "note": "ncu --set full --clock-control none, cold L2, serialised: compare shares/bytes, not absolute time",
    }
os.makedirs("profiles", exist_ok=True)
json.dump(summary, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps(summary, indent=1))
