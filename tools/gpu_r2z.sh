mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/k3_sanity.py > gpurun_out/sanitizer_k3_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_k3_$tool.txt
done
