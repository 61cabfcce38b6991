mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/kernel_times.py 26 > gpurun_out/ktimes.log 2>&1
timeout 300 python tools/kernel_times.py 26 --opt PREMAP_IN_SPLIT=1 > gpurun_out/ktimes_old.log 2>&1
