mkdir -p gpurun_out
( python tools/sweep.py 131072,524288 1 h64_tp4_rank,h64_mla_tp4_rank gpurun_out/h64_base.md
  MLRA_DEBUG_NPAD=32 python tools/sweep.py 131072,524288 1 h64_tp4_rank gpurun_out/h64_npad32.md
  MLRA_DEBUG_NPAD=16 python tools/sweep.py 131072,524288 1 h64_tp4_rank gpurun_out/h64_npad16.md
) > gpurun_out/h64_sweeps.txt 2>&1
