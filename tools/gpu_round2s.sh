mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/launches_bench.log 2>&1
for w in tp1 tp4; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlra_decode -s 2 -c 1 \
      -o gpurun_out/k2_$w python tools/step_once.py $w > gpurun_out/ncu_k2_$w.log 2>&1
done
timeout 1200 python tools/sweep.py 131072,524288,1048576,2097152 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/sweep_h64.md > gpurun_out/sweep_h64.jsonl 2>&1
timeout 900 python tools/sweep.py 4096,32768,131072 1,16,64 tp4_rank,mla_tp4_rank gpurun_out/sweep_24h.md > gpurun_out/sweep_24h.jsonl 2>&1
