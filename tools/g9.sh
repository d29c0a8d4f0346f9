set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg4_r02d python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu17.log 2>&1
