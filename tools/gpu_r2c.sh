mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_proj_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/pytest_proj.txt 2>&1
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_prefill_gpu.py tests/test_append_gpu.py -q > gpurun_out/pytest_api.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.layer_times(torch.device('cuda', 0), None)))
" > gpurun_out/layer.txt 2>&1
