set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err
timeout 300 python tools/ncu_target.py --cfg 4 --reps 4 > gpurun_out/layout_qpmajor.log 2>&1
OCPQP_BA_STAGE_MAJOR=1 timeout 300 python tools/ncu_target.py --cfg 4 --reps 4 > gpurun_out/layout_stagemajor.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-per-config --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg4_r02 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu_c4.log 2>&1
