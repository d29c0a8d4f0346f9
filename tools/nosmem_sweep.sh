# placement experiments: OCPQP_NOSMEM bit masks (workspace buffers kept in global memory)
for v in ${NOSMEM_VARIANTS:-0}; do
  OCPQP_NOSMEM=$v timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ns_$v.json 2>&1
  echo "$v $(tail -1 gpurun_out/ns_$v.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["plan"]["smem_mask"])')" >> gpurun_out/sweep.txt
done
