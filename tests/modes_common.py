"""Shared cases of the modes-beyond-speed parity tests (tests/golden/modes.npz).

The fixture was written by tests/golden/make_golden.py (solve_modes) with the
real reference; the inputs are regenerated here from the package's own seeded
generators, so nothing under /root/reference is read at test time.

Parity rules:
  * status and IPM iteration count identical;
  * flops identical, except that modes with iterative refinement may differ by
    whole refinement solves: the number of refinement corrections is decided by
    comparisons of rounding-level residual norms (ipm_core.py:341-358), so the
    difference must be a multiple of one solve's count (sum 2 nu^2 + 2 nx0^2);
  * y, pi, lam, t within 1e-8 relative -- except the absolute formulation
    (speed_abs), whose late iterates lose accuracy by cancellation in
    ``iterate_full - iterate`` (ipm_core.py:275-283): there the first iterations
    of the trace are compared and the solution only within ABS_SOL_TOL.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from conftest import random_case_qp, rel_err

MODES = [
    ("balance6", "balance", 1e-6, {}),
    ("balance8", "balance", 1e-8, {}),
    ("robust6", "robust", 1e-6, {}),
    ("sqrt8", "speed", 1e-8, {"riccati_variant": "square_root"}),
    ("abs8", "speed_abs", 1e-8, {}),
    ("sqrtbal6", "balance", 1e-6, {"riccati_variant": "square_root"}),
]
MODE_NAMES = [m for m, *_ in MODES]
SOURCES = ([f"r{s}" for s in range(11, 17)]
           + ["c0q0", "c1q1", "c1q2", "c2q0", "c3q0", "c3q1"])
HEAVY = [("c4q56", ("balance6", "sqrt8", "robust6"))]
ABS_SOL_TOL = 1e-2


def mode_arg(name):
    from paper_2003_02547_b200 import mode_preset

    for n, preset, tol, over in MODES:
        if n == name:
            return dataclasses.replace(mode_preset(preset).with_tol(tol), **over)
    raise KeyError(name)


def source_batch(name):
    from paper_2003_02547_b200 import OcpQpBatch
    from paper_2003_02547_b200.generators import make_batch

    from conftest import random_cases

    if name.startswith("r"):
        seed = int(name[1:])
        kw = dict(random_cases())[seed]
        return OcpQpBatch.from_qps([random_case_qp(seed, kw)])
    cfg, i = int(name[1]), int(name[3:])
    return make_batch(cfg, batch=1, start=i)


def solve_flops(batch):
    d = batch.dim
    f = sum(2 * int(nu) ** 2 for nu in d.nu)
    return f + (2 * int(d.nx[0]) ** 2 if int(d.nx[0]) else 0)


def check_mode_solve(out, i, g, prefix, mode, batch):
    assert int(out["status"][i]) == int(g[f"{prefix}_status"]), "status"
    it = int(g[f"{prefix}_iters"])
    assert int(out["iters"][i]) == it, "iterations"
    df = int(out["flops"][i]) - int(g[f"{prefix}_flops"])
    arg = mode_arg(mode)
    if arg.itref_corr_max > 0 or arg.itref_pred_max > 0:
        fs = solve_flops(batch)
        assert df % fs == 0 and abs(df) <= 2 * fs * max(1, it), f"flops differ by {df}"
    else:
        assert df == 0, f"flops differ by {df}"
    tol = ABS_SOL_TOL if arg.abs_form else 1e-8
    for k in ("y", "pi", "lam", "t"):
        assert rel_err(out[k][i], g[f"{prefix}_{k}"]) <= tol, k
    tr = g[f"{prefix}_trace"]
    n = min(it, 5) if arg.abs_form else it
    if n:
        np.testing.assert_allclose(out["trace"][i, :n, :4], tr[:n, :4], rtol=1e-6, atol=1e-12)
    if arg.comp_res_pred:
        res = g[f"{prefix}_res"]
        assert np.all(np.abs(out["res"][i] - res) <= 1e-8 * np.maximum(1.0, np.abs(res)))
