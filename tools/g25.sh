#!/bin/bash
# ncu capture of the generic kernel on the partially condensed config 4 (nx 60, nu 100, ng 240, N2 20)
set -u
mkdir -p gpurun_out
timeout 600 python tools/ncu_target.py --cfg 4 --reps 2 --path partial:5 > gpurun_out/partial_plain.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ipm_solve -s 1 -c 1 -o gpurun_out/prof_cfg4_partial_r02 python tools/ncu_target.py --cfg 4 --reps 2 --path partial:5 > gpurun_out/ncu_partial.log 2>&1
echo done > gpurun_out/g25_done.txt
