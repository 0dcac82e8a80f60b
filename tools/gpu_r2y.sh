mkdir -p gpurun_out
TRACE_B=1 TRACE_L=131072 timeout 300 python tools/trace_ctas.py tp4 0,1,50 > gpurun_out/trace_tp4.txt 2>&1
( python tools/step_env.py tp4; python tools/step_env.py tp4 1 131072; python tools/step_env.py tp1 ) > gpurun_out/step_env.txt 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_bench_configs_gpu.py tests/test_gqa_gpu.py -q -x > gpurun_out/pytest_y.txt 2>&1
