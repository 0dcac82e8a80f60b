#!/bin/bash
# Small-batch steps: product build vs the fused-step experiment build (grid-wide / cluster).
mkdir -p gpurun_out
for shape in "tp4 1 4096" "tp4 1 32768" "tp4 4 4096" "tp1 1 4096"; do
  cp tools/bin/var_G/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so 2>/dev/null
  python tools/step_env.py $shape >> gpurun_out/small_fuse.txt 2>&1
  cp tools/bin/var_H/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
  MLRA_FUSE_GRID=1 python tools/step_env.py $shape >> gpurun_out/small_fuse.txt 2>&1
  MLRA_FUSE_CLUSTER=1 python tools/step_env.py $shape >> gpurun_out/small_fuse.txt 2>&1
done
