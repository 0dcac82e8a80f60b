mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_ragged_gpu.py tests/test_bench_configs_gpu.py -q -x > gpurun_out/pytest_r2k.txt 2>&1
timeout 900 python tools/sweep.py 131072,524288,1048576,2097152 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/sweep_h64.md > gpurun_out/sweep_h64.jsonl 2>&1
timeout 600 python tools/sweep.py 32768,131072 1,16 tp4_rank,mla_tp4_rank gpurun_out/sweep_24h.md > gpurun_out/sweep_24h.jsonl 2>&1
