"""Time the full-condensing path on a BASELINE config (one B200):
condense_batch -> dense IPM solve (fused kernels, N = 0 form) -> expand_batch,
against the direct Riccati solve of the same batch.  CUDA events, warm.

    python tools/fcond_bench.py [--cfg 1] [--reps 20]
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.condensing import condense_batch, expand_batch
    from paper_2003_02547_b200.generators import CONFIGS, make_batch
    from paper_2003_02547_b200.solver import get_plan

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=1)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    B = a.batch or CONFIGS[a.cfg].batch
    arg = mode_preset("speed").with_tol(1e-8)
    batch = make_batch(a.cfg, batch=B).to("cuda")

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        for _ in range(a.reps):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps, out

    t_c, (cb, cmap) = timed(lambda: condense_batch(batch))
    t_s, rep = timed(lambda: solve_ocp_qp_batch(cb, arg, trace=False))
    t_e, _ = timed(lambda: expand_batch(rep, cmap, batch))
    t_d, drep = timed(lambda: solve_ocp_qp_batch(batch, arg, trace=False))
    its = rep.iterations.float().mean().item()
    out = dict(cfg=a.cfg, B=B, nv=cmap.nv, ng=int(cb.dim.ng[0]), keep_x0=cmap.keep_x0,
               condense_ms=round(t_c, 3), dense_solve_ms=round(t_s, 3), expand_ms=round(t_e, 3),
               condensed_total_ms=round(t_c + t_s + t_e, 3),
               condensed_solves_per_s=round(B / ((t_c + t_s + t_e) * 1e-3), 1),
               direct_ms=round(t_d, 3), direct_solves_per_s=round(B / (t_d * 1e-3), 1),
               dense_iters_mean=its, direct_iters_mean=drep.iterations.float().mean().item(),
               dense_plan=get_plan(cb).info())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
