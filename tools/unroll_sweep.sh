# Rebuild the config-1 team-kernel instantiation with OCPQP_NVCC_EXTRA variants and bench each.
for v in "${@:-}"; do
  touch paper_2003_02547_b200/csrc/ocpqp_fast_8_3_0_64.cu
  OCPQP_NVCC_EXTRA="$v" python -m paper_2003_02547_b200.build > /dev/null 2>&1
  r=$(timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')
  echo "[$v] $r" >> gpurun_out/unroll.txt
done
