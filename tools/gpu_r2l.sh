mkdir -p gpurun_out
rm -f gpurun_out/parity_log.jsonl
MLRA_PARITY_LOG=gpurun_out/parity_log.jsonl timeout 600 python -m pytest tests/test_bench_configs_gpu.py -q -s > gpurun_out/pytest_parity.txt 2>&1
timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_prefill_gpu.py tests/test_proj_gpu.py -q -s > gpurun_out/pytest_parity2.txt 2>&1
