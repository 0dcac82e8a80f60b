mkdir -p gpurun_out
( timeout 300 python tools/plan_uniform.py tp4 16 32768; timeout 300 python tools/plan_uniform.py tp1 16 32768; timeout 300 python tools/plan_uniform.py tp4 16 65536; timeout 300 python tools/plan_uniform.py tp4 1 131072 ) > gpurun_out/plan_uniform.txt 2>&1
