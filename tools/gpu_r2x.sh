mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_outproj_gpu.py -q -x > gpurun_out/pytest_outproj.txt 2>&1
timeout 300 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.output_side_times(torch.device('cuda', 0))))
" > gpurun_out/outproj.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python tools/outproj_once.py 16 3072 3072 > gpurun_out/sanitizer_outproj_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python tools/outproj_once.py 16 3072 3072 > gpurun_out/sanitizer_outproj_memcheck.txt 2>&1
