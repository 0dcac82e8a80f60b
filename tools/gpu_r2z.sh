mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_api_gpu.py tests/test_ragged_gpu.py tests/test_bench_configs_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/pytest_merge.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_merge.txt
( for lay in tp4 h64; do timeout 300 python tools/step_env.py $lay 1 131072; timeout 300 python tools/step_env.py $lay 1 4096; timeout 300 python tools/step_env.py $lay 16 32768; done ) > gpurun_out/step_env.txt 2>&1
