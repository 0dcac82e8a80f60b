#!/bin/bash
# Re-entry check of HEAD: GPU suite, smoke, bench line, reference arm.
mkdir -p gpurun_out
timeout 420 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "exit $?" >> gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
