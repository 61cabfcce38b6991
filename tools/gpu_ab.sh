mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "config4 or batch or small" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/batch_bench.py 4096 16 low > gpurun_out/batch.log 2>&1
timeout 300 python tools/batch_bench.py 4096 16 high >> gpurun_out/batch.log 2>&1
