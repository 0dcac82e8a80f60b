mkdir -p gpurun_out
for ks in "" 2 3 4 5 6 8; do
  if [ -z "$ks" ]; then python tools/proj_time.py; else MLRA_DEBUG_PROJ_KS=$ks python tools/proj_time.py; fi
done > gpurun_out/proj_time.txt 2>&1
timeout 900 python -m pytest tests/test_proj_gpu.py tests/test_layer_gpu.py -q > gpurun_out/pytest_proj.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:proj_gemm -s 4 -c 2 -o gpurun_out/proj python tools/proj_time.py > gpurun_out/ncu_proj.log 2>&1
