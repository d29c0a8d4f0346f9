"""Aggregate an ncu source-page SASS export by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep OBJECT.o [--top 40]

ncu's CSV source page lists per-SASS-instruction metrics without line info;
nvdisasm -g on the same object gives the SASS-address -> source-line map.  The
join prints the source lines with the most executed instructions and warp
stall samples.
"""

from __future__ import annotations

import argparse
import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("obj")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--kernel", default="k_fast_solve")
    ap.add_argument("--stall", default="Warp Stall Sampling (All Samples)",
                    help="source-page column to rank by, e.g. stall_long_sb")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    lines = raw.splitlines()
    hdr_i = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rd = csv.DictReader(io.StringIO("\n".join(lines[hdr_i:])))
    metrics = {}
    base = None
    for row in rd:
        try:
            addr = int(row["Address"], 16) if row["Address"].startswith("0x") else int(row["Address"])
        except (ValueError, KeyError):
            continue
        if base is None:
            base = addr
        addr -= base
        def f(k):
            try:
                return float(row.get(k) or 0)
            except ValueError:
                return 0.0
        metrics[addr] = (f("Instructions Executed"), f(a.stall))
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(a.obj).resolve())], cwd=td,
                       capture_output=True)
        cub = next(Path(td).glob("*.cubin"))
        dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout
    cur = None
    in_k = False
    line_of = {}
    for l in dis.splitlines():
        if l.startswith("//----") and ".text." in l:
            in_k = a.kernel in l
            continue
        if not in_k:
            continue
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m:
            cur = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    agg = defaultdict(lambda: [0.0, 0.0])
    tot_i = tot_s = 0.0
    for addr, (ins, st) in metrics.items():
        key = line_of.get(addr, ("?", 0))
        agg[key][0] += ins
        agg[key][1] += st
        tot_i += ins
        tot_s += st
    print(f"total instructions {tot_i:.3e}  stall samples {tot_s:.0f}")
    src_cache = {}
    for key, (ins, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: a.top]:
        fn, ln = key
        text = ""
        p = Path(__file__).resolve().parents[1] / "paper_2003_02547_b200" / "csrc" / fn
        if p.exists():
            src_cache.setdefault(fn, p.read_text().splitlines())
            if 0 < ln <= len(src_cache[fn]):
                text = src_cache[fn][ln - 1].strip()[:90]
        print(f"{fn}:{ln:5d}  inst {100 * ins / max(tot_i, 1):5.1f}%  stall {100 * st / max(tot_s, 1):5.1f}%  {text}")


if __name__ == "__main__":
    sys.exit(main())
