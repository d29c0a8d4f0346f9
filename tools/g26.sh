#!/bin/bash
# round-2 evidence: smoke, default bench (config 4 + per_config), reference arm, launch list, ncu --set full of the config-4 solve kernel
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu_target_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg4_r02c python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu_c4.log 2>&1
timeout 600 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 3 > gpurun_out/phases_cfg4_final.jsonl 2>&1
echo done > gpurun_out/g26_done.txt
# partial path: ncu of the generic kernel on the condensed config-4 QPs, and the dense (full condensing) lines
timeout 300 python tools/ncu_target.py --cfg 4 --reps 2 --batch 148 --path partial:5 > gpurun_out/partial_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ipm_solve -s 1 -c 1 -o gpurun_out/prof_partial_r02d python tools/ncu_target.py --cfg 4 --reps 2 --batch 148 --path partial:5 > gpurun_out/ncu_partial_d.log 2>&1
for c in 1 2; do timeout 300 python tools/fcond_bench.py --cfg $c; done > gpurun_out/fcond_bench.jsonl 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_final.log
echo done2 > gpurun_out/g26_done2.txt
