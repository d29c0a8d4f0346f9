"""Minimal profiling target: N solves of one config's batch (speed, 1e-8).

    python tools/ncu_target.py --cfg 4 [--reps 3] [--batch B] [--path ocp|partial:5]

Used under ``ncu -k regex:k_fast_solve -s <reps-1> -c 1`` so the captured
launch is a warm one (same kernel, same inputs as bench.py's timed steps).
Prints the event-timed duration of each solve.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.generators import CONFIGS, make_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--path", default="ocp")
    ap.add_argument("--mode", default="speed")
    a = ap.parse_args()
    arg = mode_preset(a.mode).with_tol(1e-8 if a.mode not in ("balance", "robust") else 1e-6)
    B = a.batch or CONFIGS[a.cfg].batch
    dev = make_batch(a.cfg, batch=B).to("cuda")
    if a.path.startswith("partial:"):
        from paper_2003_02547_b200.condensing import partial_condense_batch

        dev, _ = partial_condense_batch(dev, int(a.path.split(":")[1]))
    for r in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = solve_ocp_qp_batch(dev, arg, trace=False)
        e1.record()
        torch.cuda.synchronize()
        its = rep.iterations.cpu()
        print(f"rep {r}: {e0.elapsed_time(e1):.3f} ms, iterations mean {its.float().mean():.2f} "
              f"max {int(its.max())}", flush=True)


if __name__ == "__main__":
    main()
