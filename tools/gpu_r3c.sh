#!/bin/bash
# First-tile rule A/B: B = vote always, C = exact always, D = exact when the split has >= 16 tiles.
mkdir -p gpurun_out
for v in B C D; do
  cp tools/bin/var_$v/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
  echo "== variant $v" >> gpurun_out/k2_ab2.txt
  timeout 300 python tools/k2_time.py tp1 tp4 mla >> gpurun_out/k2_ab2.txt 2>&1
  timeout 400 python tools/sweep.py 131072,524288 1 h64_tp4_rank gpurun_out/sweep_$v.md > gpurun_out/sweep_$v.jsonl 2>&1
done
cp tools/bin/var_D/libmlra_b200.so paper_2603_02188_b200/libmlra_b200.so
