"""Closed-loop MPC throughput: B spring-chain plants in lockstep on the GPU.

    python tools/mpc_bench.py [--plants 1024] [--steps 20] [--masses 4] [--horizon 15]
                              [--mode balance] [--tol 1e-6]

Each closed-loop step is one batched warm-started solve (ocpqp_solve), the
device solution shift (ocpqp_shift_guess) and the plant update; prints one
JSON line with the per-step time (CUDA events), plant-steps/s and the warm vs
cold iteration totals (a cold pass over the same trajectory's QPs).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.mpc import MassSpringConfig, run_closed_loop_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--plants", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--masses", type=int, default=4)
    ap.add_argument("--horizon", type=int, default=15)
    ap.add_argument("--mode", default="balance")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--no-cold", action="store_true", help="warm solves only")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the warm steps")
    a = ap.parse_args()
    cfg = MassSpringConfig(masses=a.masses, horizon=a.horizon)
    rng = np.random.default_rng(0)
    M = a.masses
    x0s = np.concatenate([rng.uniform(-1.0, 1.0, (a.plants, M)), np.zeros((a.plants, M))], 1)
    arg = mode_preset(a.mode).with_tol(a.tol)
    run_closed_loop_batch(cfg, x0s, 3, arg=arg, graph=not a.eager)   # warm-up (plans, kernels)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    res = run_closed_loop_batch(cfg, x0s, a.steps, arg=arg, compare_cold=not a.no_cold,
                                graph=not a.eager)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    warm = sum(r.total_iterations for r in res)
    cold = None if a.no_cold else sum(r.total_cold_iterations for r in res)
    ok = all(all(rec.status == "Success" for rec in r.records) for r in res)
    print(json.dumps({
        "workload": f"{a.plants} spring chains M={a.masses}, N={a.horizon}, {a.steps} steps, "
                    f"{a.mode} tol {a.tol:g}, warm primal_dual + paired cold solves",
        "ms_per_step": ms / a.steps, "wall_s": wall, "includes_cold_solves": not a.no_cold,
        "cuda_graph": not a.eager,
        "plant_steps_per_s": a.plants * a.steps / (ms * 1e-3),
        "warm_iterations": warm, "cold_iterations": cold,
        "warm_over_cold": warm / cold if cold else None, "all_success": ok}))


if __name__ == "__main__":
    main()
