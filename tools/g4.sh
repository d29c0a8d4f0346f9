set -u
mkdir -p gpurun_out
timeout 300 python tools/ncu_target.py --cfg 4 --reps 3 > gpurun_out/t4.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu_r02d.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_r02d.log
timeout 300 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 2 > gpurun_out/sweep4.jsonl 2>&1
timeout 300 python tests/parity_report.py --cfg 4 --n 256 --json gpurun_out/parity4.json > gpurun_out/parity4.log 2>&1
