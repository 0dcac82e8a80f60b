mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_prefill_gpu.py -q -x -k "kernel_matches and mlra4-129" -s > gpurun_out/pytest_prefill1.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_prefill1.txt
