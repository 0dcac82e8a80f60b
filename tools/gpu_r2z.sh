mkdir -p gpurun_out
( cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02188_b200/csrc k3_trace.cu -o /tmp/k3_trace ) > gpurun_out/k3_trace.txt 2>&1
/tmp/k3_trace >> gpurun_out/k3_trace.txt 2>&1
( for i in 1 2; do timeout 300 python tools/step_env.py tp1 16 32768; timeout 300 python tools/step_env.py tp4 16 32768; done ) > gpurun_out/step_env.txt 2>&1
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_api_gpu.py tests/test_bench_configs_gpu.py tests/test_ragged_gpu.py -q -x > gpurun_out/pytest_k3.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_k3.txt
