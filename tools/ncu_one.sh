#!/bin/bash
# One full-set ncu capture of a kernel (regex $1) of the 2^LG products (after
# the warm-up launches), summarised on the box: bash tools/ncu_one.sh REGEX TAG [LG] [SKIP]
K=$1; T=$2; LG=${3:-26}; S=${4:-3}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/${T} -f python tools/prof_case.py $LG > gpurun_out/ncu_${T}.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}.ncu-rep > gpurun_out/${T}_summary.md 2>&1
python tools/ncu_lines.py gpurun_out/${T}.ncu-rep "$K" 400 0 > gpurun_out/${T}_lines.txt 2>&1
rm -f gpurun_out/${T}.ncu-rep
