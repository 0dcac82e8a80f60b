mkdir -p gpurun_out
( python tools/step_env.py tp4
  MLRA_DEBUG_RING=3,3,2 python tools/step_env.py tp4
  MLRA_DEBUG_RING=5,5,2 python tools/step_env.py tp4
  MLRA_NO_PDL=1 python tools/step_env.py tp4
  MLRA_DEBUG_RING=3,3,2 MLRA_K1_MMA=1 python tools/step_env.py tp4
) > gpurun_out/step_env.txt 2>&1
