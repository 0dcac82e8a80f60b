mkdir -p gpurun_out
( for sp in 0 1 2; do echo "spin=$sp"; MLRA_DEBUG_PF_SPIN=$sp timeout 300 python tools/prefill_time.py 1024 4096 16384; done ) > gpurun_out/prefill_time.txt 2>&1
MLRA_DEBUG_PF_SPIN=1 timeout 120 python tools/prefill_check.py mlra4 1000 > gpurun_out/prefill_dbg.txt 2>&1
