"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_target.py [--cfg 1 4] [--balance]

Runs each listed config's shaped team kernel (and the balance-mode variant
with --balance) on a few QPs -- config 4 on a shortened horizon, the same
compile-time shape and code paths (factor_big, TMA sweeps and residuals) --
and checks the result against the CPU oracle so a silent corruption fails too.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main():
    import torch

    import oracle as orc
    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.generators import make_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="*", default=[1, 4])
    ap.add_argument("--balance", action="store_true")
    a = ap.parse_args()
    shapes = {0: (1, None), 1: (4, None), 2: (2, 6), 3: (2, 6), 4: (2, 8)}
    modes = [("speed", 1e-8)] + ([("balance", 1e-6)] if a.balance else [])
    for cfg in a.cfg:
        B, N = shapes[cfg]
        batch = make_batch(cfg, batch=B, N=N)
        for mode, tol in modes:
            arg = mode_preset(mode).with_tol(tol)
            rep = solve_ocp_qp_batch(batch, arg)
            torch.cuda.synchronize()
            ref = orc.solve(batch, arg, nthreads=1, trace=False)
            ok = np.array_equal(rep.iterations.cpu().numpy(), ref["iters"])
            err = float(np.max(np.abs(rep.y.cpu().numpy() - ref["y"])))
            print(f"cfg {cfg} (B={B}, N={batch.dim.N}) {mode}: iterations match {ok}, "
                  f"max |dy| {err:.2e}", flush=True)
            assert ok and err < 1e-6


if __name__ == "__main__":
    main()
