set -u
mkdir -p gpurun_out

timeout 300 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/t12.log 2>&1
timeout 300 python tests/parity_report.py --cfg 4 --n 64 > gpurun_out/parity12.log 2>&1
timeout 300 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 2 > gpurun_out/sweep12.jsonl 2>&1
timeout 300 python tools/sweep.py --cfg 4 --batch 64 --kinds 0 --phases --reps 2 >> gpurun_out/sweep12.jsonl 2>&1
