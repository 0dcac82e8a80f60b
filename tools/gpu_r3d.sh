#!/bin/bash
# Round-2 final evidence (lean K2): GPU suite, smoke, bench + reference arm, K2 timings, h64 sweep,
# launch list of the bench command, full ncu captures of K2 (TP1, TP4 rank).
mkdir -p gpurun_out
timeout 420 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "exit $?" >> gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 300 python tools/k2_time.py tp1 tp4 mla > gpurun_out/k2_time.txt 2>&1
timeout 600 python tools/sweep.py 131072,524288,1048576,2097152 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/sweep_h64.md > gpurun_out/sweep_h64.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/launches_bench.log 2>&1
for w in tp1 tp4; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlra_decode -s 2 -c 1 \
      -o gpurun_out/k2_$w python tools/step_once.py $w > gpurun_out/ncu_k2_$w.log 2>&1
done
ls -la gpurun_out
