#!/bin/bash
# Ring depth A/B at the TP4 rank and TP1 (B = 16, 32K): K2 alone and the step.
mkdir -p gpurun_out
for ring in default 4,4,1 5,3,1 5,4,1 3,3,2 5,2,1; do
  if [ $ring = default ]; then unset MLRA_DEBUG_RING; else export MLRA_DEBUG_RING=$ring; fi
  echo "== ring $ring $(python tools/step_env.py tp4 2>&1 | grep step)" >> gpurun_out/ring_tp4.txt
done
for ring in default 5,1,1 6,1,1 4,1,1 4,2,2; do
  if [ $ring = default ]; then unset MLRA_DEBUG_RING; else export MLRA_DEBUG_RING=$ring; fi
  echo "== ring $ring $(python tools/step_env.py tp1 2>&1 | grep step)" >> gpurun_out/ring_tp4.txt
done
