mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "split_carry or option or c_demo or cpp" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python tools/kernel_times.py 18 20 22 24; timeout 300 python tools/kernel_times.py 18 20 22 24 --opt SPLIT_AGGREGATES=1; done > gpurun_out/ktimes.log 2>&1
