#!/bin/bash
# B = 2 K3 choice: auto (new rule) vs forced split-K (1) / per-branch (2).
mkdir -p gpurun_out
for shape in "tp4 2 4096" "tp4 2 8192" "tp4 2 16384" "tp4 2 32768" "tp4 2 131072" "h64 2 32768" "tp1 2 32768" "mla 2 32768"; do
  for f in auto 1 2; do
    if [ $f = auto ]; then unset MLRA_K3_FORCE; else export MLRA_K3_FORCE=$f; fi
    echo "K3=$f $(python tools/split_sweep.py $shape 2>&1 | grep step)" >> gpurun_out/k3_b2.txt
  done
done
timeout 300 python -m pytest tests/test_decode_gpu.py tests/test_api_gpu.py -q > gpurun_out/pytest_k3_b2.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_k3_b2.txt
