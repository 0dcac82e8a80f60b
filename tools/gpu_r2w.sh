mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
( python tools/step_env.py tp1; python tools/step_env.py tp1 1 131072; python tools/step_env.py tp1 64 32768 ) > gpurun_out/step_env.txt 2>&1
TRACE_B=16 TRACE_L=32768 timeout 300 python tools/trace_ctas.py tp1 0,1,50 > gpurun_out/trace_tp1.txt 2>&1
