mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref_r1g.json 2> gpurun_out/bench_ref_r1g.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1g.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 22 -c 22 -o gpurun_out/r1g_full -f python tools/prof_case.py 26 > gpurun_out/ncu_full.log 2>&1
