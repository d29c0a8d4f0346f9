set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_r02a.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_r02a.log
