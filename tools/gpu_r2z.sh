mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_outproj_gpu.py tests/test_proj_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/pytest_outproj.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_outproj.txt
( cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02188_b200/csrc outproj_trace.cu -o /tmp/outproj_trace ) > gpurun_out/op_trace.txt 2>&1
( /tmp/outproj_trace 16 3072 3072 5 0; /tmp/outproj_trace 16 3072 3072 5 1 ) >> gpurun_out/op_trace.txt 2>&1
timeout 300 python tools/outproj_time.py > gpurun_out/outproj_time.txt 2>&1
timeout 300 python tools/proj_time.py > gpurun_out/proj_time.txt 2>&1
