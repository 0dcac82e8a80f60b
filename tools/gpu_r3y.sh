#!/bin/bash
# K3 variant at the benchmarked B = 16 shapes (auto = per-branch CTAs).
mkdir -p gpurun_out
for shape in "tp4 16 32768" "tp1 16 32768" "tp4 16 131072" "h64 16 32768" "mla 16 32768" "tp4 64 32768"; do
  for f in auto 1 3; do
    if [ $f = auto ]; then unset MLRA_K3_FORCE; else export MLRA_K3_FORCE=$f; fi
    echo "K3=$f $(python tools/split_sweep.py $shape 2>&1 | grep step)" >> gpurun_out/k3_b16.txt
  done
done
