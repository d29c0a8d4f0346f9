#!/bin/bash
# round-2 check: GPU tests, default bench, reference arm, ncu capture of the partial path's solve kernel
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
timeout 600 python tools/ncu_target.py --cfg 4 --reps 2 --batch 148 --path partial:5 > gpurun_out/partial_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ipm_solve -s 1 -c 1 -o gpurun_out/prof_partial_r02 python tools/ncu_target.py --cfg 4 --reps 2 --batch 148 --path partial:5 > gpurun_out/ncu_partial.log 2>&1
cat gpurun_out/partial_plain.log
echo done
