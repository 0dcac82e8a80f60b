#!/bin/bash
# K4 A/B: E = 4-stage ring (3 primed, GEMM after the whole prime landed), F = 5 stages all primed,
# chunk-by-chunk GEMM, residual prefetched, two accumulator sets. Then the output-side tests on F.
mkdir -p gpurun_out
for pass in 1 2; do
  for v in E F; do
    cp tools/bin/var_$v/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
    echo "== pass $pass variant $v" >> gpurun_out/k4_ab.txt
    NOSIM=1 timeout 300 python tools/outproj_time.py >> gpurun_out/k4_ab.txt 2>&1
  done
done
cp tools/bin/var_F/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
timeout 300 python -m pytest tests/test_outproj_gpu.py -q > gpurun_out/pytest_outproj.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_outproj.txt
python tools/outproj_time.py > gpurun_out/k4_sim.txt 2>&1
