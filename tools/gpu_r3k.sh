#!/bin/bash
# K3 change (four MMA chains, unrolled k loop, branch sum spread over the cluster): phase trace,
# per-kernel times, the K3-touching GPU tests.
mkdir -p gpurun_out
(cd tools && ./k3_trace) > gpurun_out/k3_trace2.txt 2>&1
python tools/kernel_times.py 16 32768 > gpurun_out/kt2.txt 2>&1
timeout 400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_k3.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_k3.txt
python tools/step_env.py tp1 >> gpurun_out/kt2.txt 2>&1
