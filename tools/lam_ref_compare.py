"""Three-way lambda comparison on the QPs saved by tools/lam_diag.py (build container).

    PYTHONPATH=/root/reference/pkg/src python tools/lam_ref_compare.py gpurun_out/lam3.npz [--json out]

Runs the REAL reference (mpcqp.solve_ocp_qp, speed, tol 1e-8; and its
square-root variant) on each saved QP and reports, per QP, the relative
lambda / y / pi / t differences reference-vs-GPU, reference-vs-oracle and
reference classical-vs-square-root (the known-hard config-3 row).
"""

from __future__ import annotations

import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
sys.path.insert(0, str(ROOT / "tests"))

import mpcqp  # noqa: E402  (the reference, build container only)

from paper_2003_02547_b200.generators import make_batch  # noqa: E402


def rel(a, r):
    return float(np.max(np.abs(a - r)) / max(1.0, float(np.max(np.abs(r)))))


def main():
    from make_golden import to_ref

    d = np.load(sys.argv[1])
    cfg = int(d["cfg"])
    arg = mpcqp.mode_preset("speed").with_tol(1e-8)
    argsq = replace(arg, riccati_variant="square_root")
    rows = []
    for j, i in enumerate(d["idx"]):
        qp = to_ref(make_batch(cfg, batch=1, start=int(i)).qp(0))
        r = mpcqp.solve_ocp_qp(qp, arg)
        rs = mpcqp.solve_ocp_qp(qp, argsq)
        s = r.solution
        row = dict(qp=int(i), bad=j < int(d["nbad"]), ref_iters=r.iterations,
                   gpu_iters=int(d["gpu_iters"][j]), ora_iters=int(d["ora_iters"][j]),
                   sqrt_iters=rs.iterations)
        for k in ("lam", "y", "pi", "t"):
            ref = getattr(s, k)
            row[f"{k}_ref_gpu"] = rel(d[f"gpu_{k}"][j], ref)
            row[f"{k}_ref_ora"] = rel(d[f"ora_{k}"][j], ref)
            row[f"{k}_ref_sqrt"] = rel(getattr(rs.solution, k), ref)
            row[f"{k}_gpu_ora"] = rel(d[f"gpu_{k}"][j], d[f"ora_{k}"][j])
        rows.append(row)
        print(json.dumps(row), flush=True)
    bad = [r for r in rows if r["bad"]]
    summ = {"cfg": cfg, "qps": len(rows), "bad": len(bad)}
    for k in ("lam_ref_gpu", "lam_ref_ora", "lam_ref_sqrt", "lam_gpu_ora", "y_ref_gpu", "y_ref_ora"):
        v = np.array([r[k] for r in bad]) if bad else np.zeros(1)
        summ[k] = {"max": float(v.max()), "n_gt_1e-8": int(np.sum(v > 1e-8))}
    print(json.dumps(summ))
    if "--json" in sys.argv:
        Path(sys.argv[sys.argv.index("--json") + 1]).write_text(
            json.dumps({"summary": summ, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
