# Rebuild one team-kernel instantiation with OCPQP_MINB_THREADS variants and bench a config.
# usage: bash tools/minb_sweep.sh FILE CFG V1 V2 ...
f=$1; cfg=$2; shift 2
for v in "$@"; do
  touch paper_2003_02547_b200/csrc/$f
  OCPQP_NVCC_EXTRA="-DOCPQP_MINB_THREADS=$v" python -m paper_2003_02547_b200.build > /dev/null 2>&1
  r=$(timeout 300 python bench.py --cfg $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["plan"]["slots"])')
  echo "cfg$cfg minb_threads=$v $r" >> gpurun_out/minb.txt
done
