set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python tools/lam_diag.py > gpurun_out/lam_diag.log 2>&1
timeout 300 python tools/sweep.py --cfg 4 3 2 1 --kinds 0 --phases --reps 2 > gpurun_out/sweep_phases.jsonl 2>&1
timeout 120 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/plain4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg4_r02a python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg3_r02a python tools/ncu_target.py --cfg 3 --reps 3 > gpurun_out/ncu3.log 2>&1
echo done > gpurun_out/g1_done.txt
