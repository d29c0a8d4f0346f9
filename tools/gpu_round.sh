#!/bin/bash
# One GPU-box session: tests, benches, ncu evidence (outputs under gpurun_out/).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
for c in 2 3 4; do
  timeout 600 python bench.py --cfg $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_cfg1.json 2>&1
for m in balance sqrt speed_abs robust; do
  timeout 300 python bench.py --mode $m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mode_$m.json 2> /dev/null
done
for c in 1 2; do timeout 300 python tools/fcond_bench.py --cfg $c; done > gpurun_out/fcond_bench.jsonl 2>&1
# ncu: launch list then one full capture of the solve kernel (same command exited 0 first)
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 3 -c 1 -o gpurun_out/prof_cfg1_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo done > gpurun_out/round_done.txt
