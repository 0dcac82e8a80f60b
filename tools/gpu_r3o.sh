#!/bin/bash
# 64-head ring depth A/B (MLRA_DEBUG_RING=lat,rope,p; default 3,3,2): K2 at B = 1, 128K and 1M.
mkdir -p gpurun_out
for ring in default 3,3,1 4,2,1 4,3,1 3,4,1 2,2,2; do
  if [ $ring = default ]; then unset MLRA_DEBUG_RING; else export MLRA_DEBUG_RING=$ring; fi
  timeout 300 python tools/sweep.py 131072,1048576 1 h64_tp4_rank gpurun_out/ring_$ring.md > /dev/null 2>&1
  echo "== ring $ring" >> gpurun_out/ring.txt; grep h64 gpurun_out/ring_$ring.md >> gpurun_out/ring.txt
done
