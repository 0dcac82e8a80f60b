#!/bin/bash
# Rescale threshold A/B (MLRA_DEBUG_RESCALE_THRESHOLD; product 8): K2 alone TP1 / TP4 / MLA and
# the 64-head batch-1 K2 at 128K / 1M.
mkdir -p gpurun_out
for thr in 8 12 16; do
  echo "== thr $thr" >> gpurun_out/thr.txt
  MLRA_DEBUG_RESCALE_THRESHOLD=$thr timeout 300 python tools/k2_time.py tp1 tp4 mla >> gpurun_out/thr.txt 2>&1
  MLRA_DEBUG_RESCALE_THRESHOLD=$thr timeout 300 python tools/sweep.py 131072,1048576 1 h64_tp4_rank gpurun_out/thr_$thr.md > /dev/null 2>&1
  grep h64 gpurun_out/thr_$thr.md >> gpurun_out/thr.txt
done
