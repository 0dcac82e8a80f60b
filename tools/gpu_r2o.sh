mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python tools/prefill_time.py 1024 4096 16384 > gpurun_out/prefill_time.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_smoke_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_smoke_$tool.txt
done
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/prefill_check.py tiny 300 > gpurun_out/sanitizer_prefill_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_prefill_$tool.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/outproj_once.py 16 3072 3072 > gpurun_out/sanitizer_outproj_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_outproj_$tool.txt
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_ragged_gpu.py -q -x -k "plan_covers" > gpurun_out/sanitizer_plan_memcheck.txt 2>&1
echo "exit $?" >> gpurun_out/sanitizer_plan_memcheck.txt
