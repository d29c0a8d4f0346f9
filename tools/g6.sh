set -u
mkdir -p gpurun_out
./tools/ubench/dmma > gpurun_out/dmma.txt 2>&1
timeout 300 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/t6.log 2>&1
timeout 300 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 2 > gpurun_out/sweep6.jsonl 2>&1
timeout 300 python tools/sweep.py --cfg 4 --batch 64 --kinds 0 --phases --reps 2 >> gpurun_out/sweep6.jsonl 2>&1
