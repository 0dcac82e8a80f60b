#!/bin/bash
# K3 variant per shape for the MLA baseline (TP4 rank, 24-head and 64-head shapes).
mkdir -p gpurun_out
for shape in "mla 1 4096" "mla 2 4096" "mla 4 4096" "mla 8 4096" "mla 1 32768" "mla 2 32768" "mla 4 32768" "mla 8 32768" "mla 16 32768" "h64mla 1 131072" "h64mla 1 1048576"; do
  for f in auto 1 2 3; do
    if [ $f = auto ]; then unset MLRA_K3_FORCE; else export MLRA_K3_FORCE=$f; fi
    echo "K3=$f $(python tools/split_sweep.py $shape 2>&1 | grep step)" >> gpurun_out/k3_variants_mla.txt
  done
done
