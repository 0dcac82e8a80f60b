#!/bin/bash
# K3 variant rule (merge + head GEMM only at batch 1): GPU suite, the small-batch shapes, sweep.
mkdir -p gpurun_out
timeout 420 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_k3v.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_k3v.txt
for shape in "tp4 1 4096" "tp4 2 4096" "tp4 4 4096" "tp4 8 4096" "tp4 1 32768" "tp4 2 32768" "tp4 4 32768" "tp4 8 32768" "tp4 8 131072" "h64 1 131072" "h64 4 4096" "h64 2 32768" "tp1 4 32768"; do
  python tools/split_sweep.py $shape 2>&1 | grep step >> gpurun_out/k3v_after.txt
done
timeout 1500 python tools/sweep.py > gpurun_out/sweep_24h_k3v.jsonl 2> gpurun_out/sweep_24h_k3v.err
cp gpurun_out/sweep.md gpurun_out/sweep_24h_k3v.md
