#!/bin/bash
# generic-kernel development check: condensing / dense / mode tests, then the partial path timing
timeout 900 python -m pytest tests/test_gpu_condense.py tests/test_gpu_fcond.py tests/test_gpu_soft_cond.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -4
for b in ${BATCHES:-148 256}; do echo "batch $b"; timeout 300 python tools/ncu_target.py --cfg 4 --reps 2 --batch $b --path partial:5 | tail -1; done
