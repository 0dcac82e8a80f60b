mkdir -p gpurun_out
MLRA_PARITY_LOG=gpurun_out/parity_h64.jsonl timeout 900 python -m pytest tests/test_bench_configs_gpu.py -q -x -k "64_heads or long_context" -s > gpurun_out/pytest_h64.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_h64.txt
