#!/bin/bash
# 64 heads at B = 2-3: merge + head GEMM (3) vs per-branch CTAs (2).
mkdir -p gpurun_out
for shape in "h64 2 4096" "h64 2 8192" "h64 2 32768" "h64 2 131072" "h64 3 32768" "h64 4 32768"; do
  for f in auto 2 3; do
    if [ $f = auto ]; then unset MLRA_K3_FORCE; else export MLRA_K3_FORCE=$f; fi
    echo "K3=$f $(python tools/split_sweep.py $shape 2>&1 | grep step)" >> gpurun_out/k3_h64b2.txt
  done
done
