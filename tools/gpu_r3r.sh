#!/bin/bash
# Split-count sweep, small batches x short contexts (policy check for mlra_default_splits).
mkdir -p gpurun_out
for shape in "2 4096" "4 4096" "8 4096" "4 8192" "8 8192" "4 16384" "8 16384" "2 8192" "1 8192"; do
  set -- $shape
  def=$(( 148 / $1 ))
  python tools/split_sweep.py tp4 $1 $2 $def,48,37,33,24,16,12,8,6,4 >> gpurun_out/split_sweep2.txt 2>&1
done
python tools/split_sweep.py tp1 4 4096 37,33,16,8,4 >> gpurun_out/split_sweep2.txt 2>&1
python tools/split_sweep.py h64 4 4096 37,33,16,8,4 >> gpurun_out/split_sweep2.txt 2>&1
