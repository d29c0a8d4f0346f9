set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dense_eq.py tests/test_gpu_safety.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_dense_eq.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_dense_eq.log
