#!/bin/bash
# GPU iteration loop: parity tests, per-kernel times at 2^26, short bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/kernel_times.py 26 > gpurun_out/ktimes.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
