mkdir -p gpurun_out
timeout 300 python tools/kernel_times.py 16 32768 > gpurun_out/ktimes_b16.txt 2>&1
timeout 300 python tools/step_ab.py > gpurun_out/step_ab.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_smoke_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_smoke_$tool.txt
done
