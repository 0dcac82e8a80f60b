#!/bin/bash
# Round profile: bench line, launch list of the bench command, full ncu capture of K2 (TP1 + TP4 rank).
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/launches_bench.log 2>&1
for w in tp1 tp4; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlra_decode -s 2 -c 1 \
      -o gpurun_out/k2_$w python tools/step_once.py $w > gpurun_out/ncu_k2_$w.log 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:outproj_allreduce -s 2 -c 1 \
    -o gpurun_out/k4 python tools/outproj_once.py 16 3072 3072 > gpurun_out/ncu_k4.log 2>&1
ls -la gpurun_out
