#!/bin/bash
# Round-2 final evidence, lean K2 + the bench's K2 roofline timed right after the timed steps:
# GPU suite, smoke, bench + reference arm, launch list, K2 ncu captures, 24-head context x batch
# sweep, compute-sanitizer on the smoke step.
mkdir -p gpurun_out
timeout 420 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "exit $?" >> gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/launches_bench.log 2>&1
for w in tp1 tp4; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlra_decode -s 2 -c 1 \
      -o gpurun_out/k2_$w python tools/step_once.py $w > gpurun_out/ncu_k2_$w.log 2>&1
done
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_$tool.txt 2>&1
done
timeout 1200 python tools/sweep.py > gpurun_out/sweep_24h.jsonl 2> gpurun_out/sweep_24h.err
ls -la gpurun_out
