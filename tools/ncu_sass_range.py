"""Per-SASS-instruction view of a source-line range from an ncu capture.

    python tools/ncu_sass_range.py REPORT.ncu-rep OBJECT.o LO HI [--file ocpqp_fast.cuh]

Prints, in address order, every instruction whose line-table entry falls in
[LO, HI] of the given source file: executed warp instructions, stall samples
and the two largest stall reasons -- to see which instruction of a loop body
the warps wait on.
"""

from __future__ import annotations

import argparse
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("obj")
    ap.add_argument("lo", type=int)
    ap.add_argument("hi", type=int)
    ap.add_argument("--file", default="ocpqp_fast.cuh")
    ap.add_argument("--kernel", default="k_fast_solve")
    ap.add_argument("--min-exec", type=float, default=1.0)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    hdr_i = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[hdr_i:]))))
    reasons = [k for k in rows[0].keys() if k.startswith("stall_") and "Not Issued" not in k]
    base = None
    met = {}
    for r in rows:
        try:
            addr = int(r["Address"], 16) if r["Address"].startswith("0x") else int(r["Address"])
        except (ValueError, KeyError):
            continue
        base = addr if base is None else base
        def f(k):
            try:
                return float(r.get(k) or 0)
            except ValueError:
                return 0.0
        met[addr - base] = (f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"),
                            sorted(((f(k), k[6:]) for k in reasons), reverse=True)[:2], r.get("Source", ""))
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(a.obj).resolve())], cwd=td, capture_output=True)
        cub = next(Path(td).glob("*.cubin"))
        dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout
    cur = None
    in_k = False
    out = []
    tot_s = sum(v[1] for v in met.values())
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
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", l)
        if m and cur and cur[0] == a.file and a.lo <= cur[1] <= a.hi:
            addr = int(m.group(1), 16)
            ex, st, top, _ = met.get(addr, (0, 0, [], ""))
            if ex >= a.min_exec:
                out.append((addr, cur[1], m.group(2).strip(), ex, st, top))
    s_range = sum(o[4] for o in out)
    print(f"range {a.lo}-{a.hi}: {len(out)} instructions, {s_range:.0f} stall samples "
          f"({100 * s_range / max(tot_s, 1):.1f}% of kernel)")
    for addr, ln, ins, ex, st, top in out:
        why = ", ".join(f"{k}:{v:.0f}" for v, k in top if v > 0)
        print(f"{addr:06x} L{ln:<5d} {ex:9.0f} {st:6.0f}  {ins[:60]:60s} {why}")


if __name__ == "__main__":
    sys.exit(main())
