#!/bin/bash
# K3 variant per shape at the default split count: auto vs MLRA_K3_FORCE=1 (split-K cluster),
# 2 (per-branch combine4), 3 (merge + head GEMM).
mkdir -p gpurun_out
for shape in "tp4 1 4096" "tp4 2 4096" "tp4 4 4096" "tp4 8 4096" "tp4 1 32768" "tp4 2 32768" "tp4 8 32768" "tp4 1 131072" "tp4 8 131072" "h64 1 131072" "h64 4 4096" "h64 2 32768" "tp1 1 32768" "tp1 4 32768" "tp1 8 8192"; do
  for f in auto 1 2 3; do
    if [ $f = auto ]; then unset MLRA_K3_FORCE; else export MLRA_K3_FORCE=$f; fi
    echo "K3=$f $(python tools/split_sweep.py $shape 2>&1 | grep step)" >> gpurun_out/k3_variants.txt
  done
done
