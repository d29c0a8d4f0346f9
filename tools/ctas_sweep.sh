# Bench a config with the resident CTAs per SM capped (OCPQP_CTAS_PER_SM).
# usage: bash tools/ctas_sweep.sh CFG V1 V2 ...
cfg=$1; shift
for v in "$@"; do
  r=$(OCPQP_CTAS_PER_SM=$v timeout 300 python bench.py --cfg $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["plan"]["slots"])')
  echo "cfg$cfg ctas_per_sm=$v $r" >> gpurun_out/ctas.txt
done
