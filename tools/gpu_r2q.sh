mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_bench_configs_gpu.py tests/test_ragged_gpu.py -q -x > gpurun_out/pytest_q.txt 2>&1
timeout 900 python tools/sweep.py 131072,524288 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/sweep_h64_q.md > /dev/null 2>&1
timeout 900 python tools/sweep.py 32768,131072 1 tp4_rank,mla_tp4_rank gpurun_out/sweep_24h_q.md > /dev/null 2>&1
