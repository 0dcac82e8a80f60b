#!/bin/bash
# Split-count sweep at small batches (the default takes one wave: min(148 / B, tiles)).
mkdir -p gpurun_out
python tools/split_sweep.py tp4 1 4096 33,24,16,12,8,6,4 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp4 1 32768 148,128,96,74,64,48,32 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp4 1 131072 148,128,96,74 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp4 4 4096 33,24,16,8 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp4 4 32768 37,32,24,16 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp4 16 4096 9,8,6,4,2 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp4 16 32768 9,8 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py tp1 1 4096 33,16,8,4 >> gpurun_out/split_sweep.txt 2>&1
python tools/split_sweep.py h64 1 131072 148,128,96,74 >> gpurun_out/split_sweep.txt 2>&1
