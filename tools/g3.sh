set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_r02c.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_r02c.log
start=$(date +%s)
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s" >> gpurun_out/bench_r02b.err
