#!/bin/bash
# sanitizers (one tool at a time), cfg4 phase breakdown, layout experiment, cfg4/cfg3 ncu captures
set -u
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py --cfg 1 4 --balance > gpurun_out/san/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san/$tool.log
done
timeout 600 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 3 > gpurun_out/phases_cfg4.jsonl 2>&1
timeout 600 python tools/sweep.py --cfg 1 3 --kinds 0 --phases --reps 3 > gpurun_out/phases_cfg13.jsonl 2>&1
timeout 300 python tools/ncu_target.py --cfg 4 --reps 4 > gpurun_out/layout_qpmajor.log 2>&1
OCPQP_BA_STAGE_MAJOR=1 timeout 300 python tools/ncu_target.py --cfg 4 --reps 4 > gpurun_out/layout_stagemajor.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg4_r02b python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu_c4.log 2>&1
OCPQP_BA_STAGE_MAJOR=1 timeout 900 ncu --set full --clock-control none -k regex:k_fast_solve -s 2 -c 1 -o gpurun_out/prof_cfg4_stagemajor_r02 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/ncu_c4sm.log 2>&1
echo done > gpurun_out/g24_done.txt
