#!/bin/bash
# K4 A/B: E = round-2 K4, G = 5 stages all primed + A loads batched in registers; G with KS = 6.
mkdir -p gpurun_out
for v in E G; do
  cp tools/bin/var_$v/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
  echo "== variant $v" >> gpurun_out/k4_ab2.txt
  NOSIM=1 timeout 300 python tools/outproj_time.py >> gpurun_out/k4_ab2.txt 2>&1
done
echo "== variant G, KS<=6" >> gpurun_out/k4_ab2.txt
MLRA_DEBUG_OUTPROJ_KS=6 NOSIM=1 timeout 300 python tools/outproj_time.py >> gpurun_out/k4_ab2.txt 2>&1
echo "== variant G, KS<=4" >> gpurun_out/k4_ab2.txt
MLRA_DEBUG_OUTPROJ_KS=4 NOSIM=1 timeout 300 python tools/outproj_time.py >> gpurun_out/k4_ab2.txt 2>&1
timeout 300 python -m pytest tests/test_outproj_gpu.py -q > gpurun_out/pytest_outproj2.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_outproj2.txt
