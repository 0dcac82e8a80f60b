#!/bin/bash
# Fused-step parts at the TP4 rank (B = 16, 32K): product build vs the experiment build with the
# grid-wide fused K3 only (MLRA_FUSE_PARTS=combine), K1 only, and both.
mkdir -p gpurun_out
python tools/step_env.py tp4 >> gpurun_out/fuse_parts.txt 2>&1
cp tools/bin/var_H/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
python tools/step_env.py tp4 >> gpurun_out/fuse_parts.txt 2>&1
MLRA_FUSE_GRID=1 MLRA_FUSE_PARTS=combine python tools/step_env.py tp4 >> gpurun_out/fuse_parts.txt 2>&1
MLRA_FUSE_GRID=1 MLRA_FUSE_PARTS=absorb python tools/step_env.py tp4 >> gpurun_out/fuse_parts.txt 2>&1
MLRA_FUSE_GRID=1 python tools/step_env.py tp4 >> gpurun_out/fuse_parts.txt 2>&1
MLRA_FUSE_GRID=1 MLRA_FUSE_PARTS=combine python tools/step_env.py tp1 >> gpurun_out/fuse_parts.txt 2>&1
MLRA_FUSE_GRID=1 MLRA_FUSE_PARTS=combine python tools/step_env.py h64 1 131072 >> gpurun_out/fuse_parts.txt 2>&1
python tools/step_env.py h64 1 131072 >> gpurun_out/fuse_parts.txt 2>&1
