mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:merge_splits -s 1 -c 1 -f -o gpurun_out/k3m python tools/b1_launches.py h64_128k > gpurun_out/ncu_k3m.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:head_gemm -s 1 -c 1 -f -o gpurun_out/k3g python tools/b1_launches.py h64_128k > gpurun_out/ncu_k3g.log 2>&1
