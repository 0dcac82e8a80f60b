mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_api_gpu.py tests/test_ragged_gpu.py tests/test_gqa_gpu.py -q -x > gpurun_out/pytest_merge.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_merge.txt
timeout 900 python tools/sweep.py 4096,131072 1,16 tp4_rank,h64_tp4_rank,h64_mla_tp4_rank gpurun_out/sweep_merge.md > gpurun_out/sweep_merge.log 2>&1
