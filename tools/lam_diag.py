"""Config-3 lambda parity diagnosis (GPU box side).

    python tools/lam_diag.py [--cfg 3] [--n 512] [--thr 1e-9] [--out gpurun_out/lam3.npz]

Solves the config's batch on the GPU and with the C oracle, and saves -- for
every QP whose lambda differs by more than --thr (relative, as the parity
metric) plus a few control QPs -- the QP index and the GPU and oracle
solutions (y, pi, lam, t, status, iterations, final residuals).  The real
reference is then run on those QPs in the build container
(tools/lam_ref_compare.py) for the three-way comparison.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def rel_err(a, r):
    return np.max(np.abs(a - r), axis=1) / np.maximum(1.0, np.max(np.abs(r), axis=1))


def main():
    import torch

    import oracle as orc
    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.generators import make_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--thr", type=float, default=1e-9)
    ap.add_argument("--out", default="gpurun_out/lam3.npz")
    a = ap.parse_args()
    arg = mode_preset("speed").with_tol(1e-8)
    batch = make_batch(a.cfg, batch=a.n)
    rep = solve_ocp_qp_batch(batch.to("cuda"), arg)
    torch.cuda.synchronize()
    ref = orc.solve(batch, arg, trace=False)
    g = {k: getattr(rep, k).cpu().numpy() for k in ("y", "pi", "lam", "t")}
    e = {k: rel_err(g[k], ref[k]) for k in g}
    bad = np.flatnonzero(e["lam"] > a.thr)
    ctrl = np.setdiff1d(np.arange(min(4, a.n)), bad)
    idx = np.concatenate([bad, ctrl]).astype(np.int64)
    out = dict(idx=idx, nbad=len(bad), cfg=a.cfg,
               gpu_status=rep.status_code.cpu().numpy()[idx], gpu_iters=rep.iterations.cpu().numpy()[idx],
               gpu_res=rep.res.cpu().numpy()[idx],
               ora_status=ref["status"][idx], ora_iters=ref["iters"][idx], ora_res=ref["res"][idx])
    for k in g:
        out[f"gpu_{k}"] = g[k][idx]
        out[f"ora_{k}"] = ref[k][idx]
        out[f"err_{k}_all"] = e[k]
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    np.savez(a.out, **out)
    print(f"cfg {a.cfg}: {len(bad)} / {a.n} QPs with lam err > {a.thr:g}; max lam err "
          f"{e['lam'].max():.3e}; saved {len(idx)} QPs to {a.out}")


if __name__ == "__main__":
    main()
