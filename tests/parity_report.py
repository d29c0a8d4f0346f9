"""GPU-vs-oracle parity report over the five configs (run on a GPU box).

    python tests/parity_report.py [--cfg 1 2 3 4] [--n 64] [--mode speed|balance|...]
                                  [--tol T] [--json out.json]

For each config: solve n QPs on the GPU (fused kernel) and with the CPU oracle
(all host cores), then report status/iteration mismatches and the max
relative error ||x_gpu - x_ref||_inf / max(1, ||x_ref||_inf) of y, pi, lam, t
and of the final residual norms.  Also times the GPU solve.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def rel_err(a, r):
    scale = np.maximum(1.0, np.max(np.abs(r), axis=1))
    return np.max(np.abs(a - r), axis=1) / scale


def main():
    import torch

    import oracle as orc
    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.generators import CONFIGS, make_batch
    from paper_2003_02547_b200.solver import get_plan

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="*", default=[0, 1, 2, 3, 4])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--json", default=None)
    ap.add_argument("--mode", default="speed")
    ap.add_argument("--tol", type=float, default=None)
    a = ap.parse_args()
    tol = a.tol if a.tol is not None else (1e-6 if a.mode in ("balance", "robust") else 1e-8)
    arg = mode_preset(a.mode).with_tol(tol)
    report = {}
    for cfg in a.cfg:
        n = min(a.n, CONFIGS[cfg].batch)
        t0 = time.time()
        batch = make_batch(cfg, batch=n)
        tg = time.time() - t0
        dev = batch.to("cuda")
        rep = solve_ocp_qp_batch(dev, arg)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        rep = solve_ocp_qp_batch(dev, arg)
        s1.record()
        torch.cuda.synchronize()
        gms = s0.elapsed_time(s1)
        t0 = time.time()
        ref = orc.solve(batch, arg)
        cpu_s = time.time() - t0
        st = rep.status_code.cpu().numpy()
        its = rep.iterations.cpu().numpy()
        r = dict(n=n, gen_s=round(tg, 2), gpu_ms=round(gms, 3), cpu_s=round(cpu_s, 3),
                 plan=get_plan(dev).info(),
                 status_mismatch=int(np.sum(st != ref["status"])),
                 iter_mismatch=int(np.sum(its != ref["iters"])),
                 iters=[int(its.min()), float(its.mean()), int(its.max())],
                 status_counts={int(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))})
        for key in ("y", "pi", "lam", "t"):
            e = rel_err(getattr(rep, key).cpu().numpy(), ref[key])
            r[f"err_{key}"] = float(e.max())
            r[f"pass_{key}"] = int(np.sum(e <= 1e-8))
        res = rep.res.cpu().numpy()
        r["err_res"] = float(np.max(np.abs(res - ref["res"]) / np.maximum(1.0, np.abs(ref["res"]))))
        flo = rep.flops.cpu().numpy()
        r["flops_mismatch"] = int(np.sum(flo != ref["flops"]))
        r["mode"], r["tol"] = a.mode, tol
        bad = np.flatnonzero((st != ref["status"]) | (its != ref["iters"]))
        r["bad_idx"] = bad[:10].tolist()
        report[cfg] = r
        print(cfg, json.dumps(r), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
