#!/bin/bash
# cfg4 development check: parity tests touching the BIG kernel, then phase breakdowns
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_condense.py -q -m gpu -x -k "config4 or goldens or cfg4 or partial" -p no:cacheprovider 2>&1 | tail -5
for b in ${BATCHES:-256 148}; do timeout 300 python tools/sweep.py --cfg 4 --kinds 0 --phases --reps 3 --batch $b; done > gpurun_out/${TAG:-s}_phases.jsonl 2>&1
python - <<'P'
import json,os
for l in open('gpurun_out/%s_phases.jsonl' % os.environ.get('TAG','s')):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['B'], round(d['best_ms'],2), d['iters'], {k:(round(v/1000) if isinstance(v,(int,float)) else v) for k,v in (d.get('cycles_per_iter') or {}).items()})
P
