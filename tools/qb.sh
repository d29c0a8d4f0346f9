#!/bin/bash
# quick rebuild of selected shaped-kernel translation units + relink (development loop);
# usage: tools/qb.sh 60_20_0_256 [more stems...]; extra nvcc flags in OCPQP_NVCC_EXTRA
set -e
cd "$(dirname "$0")/.."
for s in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas=-v $OCPQP_NVCC_EXTRA \
    -c paper_2003_02547_b200/csrc/ocpqp_fast_$s.cu -o build/obj/ocpqp_fast_$s.o 2>&1 | grep -E "error|spill|registers" | head -20 &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2003_02547_b200/_lib/libocpqp_b200.so build/obj/*.o
echo linked
