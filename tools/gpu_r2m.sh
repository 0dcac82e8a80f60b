mkdir -p gpurun_out
( for e in "" "MLRA_K3_PDL=1"; do
    for a in "tp4 16 32768" "tp1 16 32768" "tp4 1 131072" "tp4 16 65536"; do env $e python tools/step_env.py $a; done
  done ) > gpurun_out/step_env.txt 2>&1
MLRA_K3_PDL=1 timeout 600 python -m pytest tests/test_bench_configs_gpu.py tests/test_api_gpu.py tests/test_bench_multirank_gpu.py tests/test_allreduce_gpu.py -q -x > gpurun_out/pytest_k3pdl.txt 2>&1
