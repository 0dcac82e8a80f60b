mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_all.txt
