#!/bin/bash
# K3 rule by batch size: GPU suite, auto-variant spot checks (MLA + MLRA-4), MLA sweep refresh.
mkdir -p gpurun_out
timeout 420 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_k3v2.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_k3v2.txt
for shape in "mla 1 4096" "mla 2 4096" "mla 4 4096" "mla 8 4096" "mla 1 32768" "mla 2 32768" "mla 4 32768" "mla 8 32768" "mla 16 32768" "h64mla 1 131072" "tp4 1 4096" "tp4 2 4096" "tp4 4 4096" "tp4 8 4096" "tp4 1 32768" "tp4 2 32768" "tp4 8 32768" "h64 1 131072" "h64 4 4096" "tp1 1 32768" "tp1 4 32768"; do
  python tools/split_sweep.py $shape 2>&1 | grep step >> gpurun_out/k3v2_after.txt
done
timeout 1500 python tools/sweep.py 4096,8192,16384,32768,65536,131072 1,4,16,64 mla_tp4_rank gpurun_out/sweep_mla2.md > gpurun_out/sweep_mla2.jsonl 2> gpurun_out/sweep_mla2.err
