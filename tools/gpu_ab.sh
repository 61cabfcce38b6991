mkdir -p gpurun_out
timeout 300 python tools/dbg_case.py 4748529 105078 > gpurun_out/dbg.log 2>&1
timeout 1500 python tools/random_sizes.py 200 9 > gpurun_out/random_sizes.log 2>&1
timeout 600 python tools/shape_sweep.py 120 > gpurun_out/shape_sweep.log 2>&1
