#!/bin/bash
# Round measurement: GPU tests, smoke, bench (both arms), ncu launch list and
# one full-set capture of a 2^26 full/low/high product sequence.
# usage: bash tools/round_measure.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 400 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 16 -c 16 -o gpurun_out/${T}_full -f python tools/prof_case.py 26 > gpurun_out/ncu_full_$T.log 2>&1
# summaries on the box (the full report exceeds what gpurun brings back)
python tools/ncu_summary.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_ncu_full.md 2>&1
python tools/ncu_traffic.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_traffic.json 2>&1
for k in k_mid_4096 k_f1d_ct k_ilast_ct k_carry_runs k_zsplit; do
  python tools/ncu_lines.py gpurun_out/${T}_full.ncu-rep "$k" 25 0 > gpurun_out/${T}_lines_$k.txt 2>&1
done
rm -f gpurun_out/${T}_full.ncu-rep
