#!/bin/bash
# ncu --set full captures: K2 at the paper's 64-head shape (B = 1, 1M) and K3 at TP1 (B = 16, 32K).
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlra_decode -s 2 -c 1 \
    -o gpurun_out/k2_h64 python tools/step_once_h64.py > gpurun_out/ncu_k2_h64.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:combine4 -s 2 -c 1 \
    -o gpurun_out/k3_tp1 python tools/step_once.py tp1 > gpurun_out/ncu_k3_tp1.log 2>&1
ls -la gpurun_out/*.ncu-rep
