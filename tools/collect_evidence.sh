#!/bin/bash
# copy the outputs of tools/g26.sh from gpurun_out/ into profiles/ (round-2 names) and refresh the ncu records
set -e
cd "$(dirname "$0")/.."
cp gpurun_out/bench_r02.json profiles/r02_bench_cfg4_default.json
cp gpurun_out/bench_ref_r02.json profiles/r02_bench_reference_cfg4.json
cp gpurun_out/launches_cfg4.csv profiles/r02_launches_cfg4.csv
cp gpurun_out/phases_cfg4_final.jsonl profiles/r02_phases_cfg4.jsonl
cp gpurun_out/pytest_gpu_final.log profiles/r02_pytest_gpu.log
cp gpurun_out/fcond_bench.jsonl profiles/r02_fcond_bench.jsonl
python tools/ncu_summary.py gpurun_out/prof_cfg4_r02c.ncu-rep profiles/r02_ncu_cfg4_summary.json --traffic profiles/ncu_traffic.json --key cfg4 > /dev/null
python tools/ncu_summary.py gpurun_out/prof_partial_r02d.ncu-rep profiles/r02_ncu_partial_summary.json > /dev/null
python tools/ncu_lines.py gpurun_out/prof_cfg4_r02c.ncu-rep build/obj/ocpqp_fast_60_20_0_256.o --top 40 > profiles/r02_ncu_cfg4_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_partial_r02d.ncu-rep build/obj/ocpqp_ipm.o --kernel k_ipm_solve --top 40 > profiles/r02_ncu_partial_lines.txt 2>&1
python - <<'P'
import csv,collections,json
rows=list(csv.reader(open('profiles/r02_launches_cfg4.csv')))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[hdr+2:]:
    if len(r)<10: continue
    try: v=float(r[-1].replace(',',''))
    except ValueError: continue
    k=r[4].split('(')[0]; agg[k][0]+=1; agg[k][1]+=v
tot=sum(v[1] for v in agg.values())
out={k:{"launches":v[0],"total_ns":v[1],"share":v[1]/tot} for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])}
json.dump({"command":"python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config (ncu --metrics gpu__time_duration.sum --clock-control none)","kernels":out}, open('profiles/r02_launches_cfg4_summary.json','w'), indent=1)
d=json.load(open('profiles/r02_bench_cfg4_default.json'))
print('cfg4', round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), 'ric', round(d['roofline']['riccati']['frac'],4), 'e2e', round(d['e2e']['value'],1), 'cpu', round(d['cpu_baseline']['value'],1))
for k,v in d['per_config'].items(): print(k, round(v['value'],1), round(v['ms_per_step'],3), round(v['roofline']['frac'],4), 'e2e', round(v.get('e2e',{}).get('value',0),1), 'cpu', round(v.get('cpu_baseline',{}).get('value',0),1), v.get('stage_ms'))
print('ref', json.load(open('profiles/r02_bench_reference_cfg4.json'))['value'])
s=json.load(open('profiles/r02_ncu_cfg4_summary.json'))
print('ncu', s['gpu__time_duration.sum'], s['dram__bytes_read.sum'], s['dram__bytes_write.sum'], s['stall_cycles_per_issue'])
print(open('profiles/ncu_traffic.json').read())
P
