"""Per-source-line stall / instruction totals from an ncu report (cuda,sass view).

    python tools/ncu_srclines.py REPORT.ncu-rep [--top 40] [--file ocpqp_fast.cuh]

Uses ncu's own source correlation (kernels compiled with -lineinfo, captured
with --import-source on), so the report alone is enough (no object file).
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--file", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = []
    cur_file = ""
    hdr = None
    for line in raw.splitlines():
        if line.startswith('"File Path"'):
            cur_file = next(csv.reader([line]))[1].split("/")[-1]
            continue
        if line.startswith('"Line No"'):
            hdr = next(csv.reader([line]))
            continue
        if hdr is None or not line.startswith('"') or line.startswith('""'):
            continue
        rec = next(csv.reader(io.StringIO(line)))
        if len(rec) < len(hdr):
            continue
        d = dict(zip(hdr, rec))
        try:
            st = float(d["Warp Stall Sampling (All Samples)"] or 0)
            ie = float(d["Instructions Executed"] or 0)
        except ValueError:
            continue
        if a.file and a.file not in cur_file:
            continue
        rows.append((st, ie, cur_file, d["Line No"], d["Source"].strip()))
    tot_s = sum(r[0] for r in rows) or 1.0
    tot_i = sum(r[1] for r in rows) or 1.0
    print(f"stall samples {tot_s:.3e}  instructions {tot_i:.3e}")
    for st, ie, f, ln, src in sorted(rows, reverse=True)[: a.top]:
        print(f"{f}:{ln:>5} stall {100 * st / tot_s:5.1f}%  inst {100 * ie / tot_i:5.1f}%  {src[:90]}")


if __name__ == "__main__":
    main()
