mkdir -p gpurun_out
timeout 600 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
for _ in range(2): print(json.dumps(bench.ragged_times(torch.device('cuda', 0), None)))
" > gpurun_out/ragged.txt 2>&1
