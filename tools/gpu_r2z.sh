mkdir -p gpurun_out
timeout 1500 python tools/sweep.py 4096,32768,131072 1,16,64 tp4_rank,mla_tp4_rank gpurun_out/r2_sweep_24h.md > gpurun_out/sweep24.log 2>&1
timeout 1500 python tools/sweep.py 131072,524288,1048576,2097152 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/r2_sweep_h64_b1_long.md > gpurun_out/sweep64.log 2>&1
