#!/bin/bash
# A/B of the K2 build variants (tools/bin/var_*): A = fused-step code compiled in (round-2 state),
# B = lean K2, C = lean + round-1 first-tile rule. K2 alone, bench-style graphs, 2 passes.
mkdir -p gpurun_out
for pass in 1 2; do
  for v in A B C; do
    cp tools/bin/var_$v/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
    echo "== pass $pass variant $v" >> gpurun_out/k2_ab.txt
    timeout 300 python tools/k2_time.py tp1 tp4 mla >> gpurun_out/k2_ab.txt 2>&1
  done
done
cp tools/bin/var_B/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
timeout 600 python bench.py --no-cpu > gpurun_out/bench_B.json 2> gpurun_out/bench_B.err
