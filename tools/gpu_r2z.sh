mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_append_gpu.py tests/test_proj_gpu.py -q -x > gpurun_out/pytest_layer.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_layer.txt
timeout 600 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
for _ in range(2): print(json.dumps(bench.layer_times(torch.device('cuda', 0), None)))
" > gpurun_out/layer.txt 2>&1
MLRA_NO_PDL=1 timeout 600 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.layer_times(torch.device('cuda', 0), None)))
" >> gpurun_out/layer.txt 2>&1
