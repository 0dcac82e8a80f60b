#!/bin/bash
# K2 with 4 softmax groups at 64 heads (608 threads): GPU suite, 64-head sweep, K2 timings.
mkdir -p gpurun_out
timeout 420 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_g4.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_g4.txt
timeout 600 python tools/sweep.py 131072,524288,1048576,2097152 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/sweep_h64_g4.md > gpurun_out/sweep_h64_g4.jsonl 2>&1
timeout 300 python tools/k2_time.py tp1 tp4 mla > gpurun_out/k2_time_g4.txt 2>&1
python tools/kernel_times.py 16 32768 > gpurun_out/kt_g4.txt 2>&1
