mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/launches_bench.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 1 -c 1 -o gpurun_out/k6 python tools/prefill_once.py 4096 > gpurun_out/ncu_k6.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:proj_gemm -s 4 -c 2 -o gpurun_out/proj python tools/proj_time.py > gpurun_out/ncu_proj.log 2>&1
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python tools/prefill_check.py tiny 300 > gpurun_out/sanitizer_prefill_memcheck.txt 2>&1
timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python tools/prefill_check.py tiny 300 > gpurun_out/sanitizer_prefill_racecheck.txt 2>&1
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_proj_gpu.py -q -x -k "golden and tiny" > gpurun_out/sanitizer_proj_memcheck.txt 2>&1
