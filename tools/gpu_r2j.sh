mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ragged_gpu.py tests/test_prefill_gpu.py tests/test_bench_configs_gpu.py -q -x > gpurun_out/pytest_ragged.txt 2>&1
timeout 300 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.ragged_times(torch.device('cuda', 0), None)))
" > gpurun_out/ragged.txt 2>&1
timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python tools/prefill_check.py tiny 300 > gpurun_out/sanitizer_prefill_racecheck.txt 2>&1
CUDA_MODULE_LOADING=EAGER timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python tools/prefill_check.py tiny 300 > gpurun_out/sanitizer_prefill_memcheck.txt 2>&1
timeout 300 python tools/step_env.py tp4 > gpurun_out/step_env.txt 2>&1
