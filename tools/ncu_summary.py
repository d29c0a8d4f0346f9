"""Summarise one ncu --set full capture (raw page) into profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json [--traffic profiles/ncu_traffic.json --key cfg1]

Writes the duration, DRAM traffic, throughput / pipe utilisation, occupancy
and the warp-stall breakdown (cycles per issued instruction) of the captured
kernel; optionally records its DRAM bytes per launch in the traffic file that
bench.py reads for roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic")
    ap.add_argument("--key")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {hdr[i]: (vals[i], units[i]) for i in range(len(hdr))}
    out = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
    for k in KEYS:
        if k in d:
            out[k] = [d[k][0], d[k][1]]
    stalls = {}
    for k, (v, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
            try:
                stalls[name] = float(v.replace(",", ""))
            except ValueError:
                pass
    out["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:12])
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    if a.traffic and a.key:
        def num(k):
            v, u = d[k]
            x = float(v.replace(",", ""))
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        try:
            tr = json.load(open(a.traffic))
        except (OSError, ValueError):
            tr = {}
        sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
        from bench import kernel_source_hash   # ties the record to the kernel sources

        tr[a.key] = {"dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                     "duration_ms": num("gpu__time_duration.sum") / 1e6 if d["gpu__time_duration.sum"][1] == "ns"
                     else float(d["gpu__time_duration.sum"][0].replace(",", "")),
                     "source": a.report.split("/")[-1], "src_hash": kernel_source_hash()}
        json.dump(tr, open(a.traffic, "w"), indent=1)
    print(json.dumps(out)[:400])


if __name__ == "__main__":
    sys.exit(main())
