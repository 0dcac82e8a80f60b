#!/bin/bash
# K3 experiment: FMA up-projection for 4 sequences per CTA too (no mma.sync).
mkdir -p gpurun_out
(cd tools && ./k3_trace) > gpurun_out/k3_trace3.txt 2>&1
python tools/kernel_times.py 16 32768 > gpurun_out/kt3.txt 2>&1
python tools/step_env.py tp1 >> gpurun_out/kt3.txt 2>&1
