mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
( python tools/step_env.py tp4; python tools/step_env.py tp1; python tools/step_env.py tp4 1 131072 ) > gpurun_out/step_env.txt 2>&1
TRACE_B=1 TRACE_L=131072 timeout 300 python tools/trace_ctas.py h64 0,1,50 > gpurun_out/trace_h64.txt 2>&1
timeout 900 python tools/sweep.py 131072,524288 1 h64_tp4_rank gpurun_out/sweep_h64_r.md > /dev/null 2>&1
