set -u
mkdir -p gpurun_out
timeout 300 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/t17.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_r02g.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_r02g.log
timeout 300 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 2 > gpurun_out/sweep17.jsonl 2>&1
timeout 300 python tools/sweep.py --cfg 4 --batch 64 --kinds 0 --phases --reps 2 >> gpurun_out/sweep17.jsonl 2>&1
