mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prefill_launches.csv python tools/prefill_once.py 4096 > gpurun_out/prefill_launches.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:prefill_attention -s 1 -c 1 -o gpurun_out/k6 python tools/prefill_once.py 4096 > gpurun_out/ncu_k6.log 2>&1
