mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_proj_gpu.py tests/test_layer_gpu.py tests/test_api_gpu.py -q -x > gpurun_out/pytest_t.txt 2>&1
python tools/proj_time.py > gpurun_out/proj_time.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 300 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.layer_times(torch.device('cuda', 0), None)))
" > gpurun_out/layer.txt 2>&1
