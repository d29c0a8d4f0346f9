"""Time the fused solve for each config and kernel kind (device-resident batch).

    python tools/sweep.py [--cfg 1 2 3 4] [--kinds 0 1] [--batch B] [--reps 3]

Prints one JSON line per (config, kernel): plan info, best/median ms per batch
solve, solves/s, iteration stats.  Kernel kind is selected through the plan's
environment override OCPQP_KIND (0 team kernel, 1 row kernel; "g" = generic).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200 import solver as S
    from paper_2003_02547_b200.generators import CONFIGS, make_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--kinds", nargs="*", default=["0", "1"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--env", nargs="*", default=[])
    ap.add_argument("--phases", action="store_true")
    a = ap.parse_args()
    for kv in a.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    arg = mode_preset("speed").with_tol(1e-8)
    for cfg in a.cfg:
        B = a.batch or CONFIGS[cfg].batch
        t0 = time.time()
        batch = make_batch(cfg, batch=B).to("cuda")
        tg = time.time() - t0
        for kind in a.kinds:
            os.environ.pop("OCPQP_KIND", None)
            os.environ.pop("OCPQP_GENERIC", None)
            if kind == "g":
                os.environ["OCPQP_GENERIC"] = "1"
            else:
                os.environ["OCPQP_KIND"] = kind
            S._PLANS.clear()
            try:
                rep = solve_ocp_qp_batch(batch, arg, trace=False)
                torch.cuda.synchronize()
            except Exception as exc:  # report and continue
                print(json.dumps({"cfg": cfg, "kind": kind, "error": str(exc)[:200]}), flush=True)
                continue
            ts = []
            for _ in range(a.reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                rep = solve_ocp_qp_batch(batch, arg, trace=False)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            its = rep.iterations.cpu().numpy()
            info = S.get_plan(batch).info()
            phases = None
            if a.phases and kind != "g":
                dbg = torch.zeros((B, 24), dtype=torch.int64, device="cuda")
                solve_ocp_qp_batch(batch, arg, trace=False, phase_debug=dbg)
                torch.cuda.synchronize()
                solve_ocp_qp_batch(batch, arg, trace=False)  # switch instrumentation off
                ph = dbg.cpu().numpy().astype(float)
                n_it = np.maximum(ph[:, 6], 1)
                names = {0: "res", 1: "factor_rest", 2: "aff_rest", 3: "dir_rest", 4: "step",
                         8: "f_T1", 9: "f_G", 10: "f_chol", 11: "f_K", 12: "f_P",
                         13: "s_pre_post", 14: "s_bwd", 15: "s_fwd"}
                phases = {nm: round(float(np.mean(ph[:, i] / n_it))) for i, nm in names.items()}
                for x in range(8):   # free diagnostic slots (OCPQP_XDIAG builds)
                    if ph[:, 16 + x].any():
                        phases[f"x{x}"] = round(float(np.mean(ph[:, 16 + x] / n_it)))
                phases["total_per_iter"] = float(np.mean(ph[:, 5] / n_it))
                phases["max_total_cycles"] = float(ph[:, 5].max())
            print(json.dumps({"cfg": cfg, "kind": kind, "B": B, "gen_s": round(tg, 1),
                              "best_ms": min(ts), "median_ms": float(np.median(ts)),
                              "solves_per_s": B / (min(ts) * 1e-3),
                              "iters": [int(its.min()), float(its.mean()), int(its.max())],
                              "cycles_per_iter": phases, "plan": info}), flush=True)


if __name__ == "__main__":
    main()
