"""CPU restatement of the closed-loop MPC driver (TEST INFRASTRUCTURE ONLY).

numpy restatement of mass_spring._shift_guess (mass_spring.py:152-195) and
run_closed_loop (mass_spring.py:222-273) over the C oracle's warm-started
solve (oracle.py).  Pinned by tests/test_mpc_oracle.py to the reference's
trajectories in tests/golden/closed_loop.npz; used only by tests/ as the
checker of paper_2003_02547_b200.mpc.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

import oracle as orc


def shift_guess(batch, sol):
    """One QP (batch.B == 1): sol = dict/tuple of (y, pi, lam, t) 1-d arrays."""
    from paper_2003_02547_b200.layout import QpSolution

    lay = batch.layout
    d = batch.dim
    N = d.N
    y, pi, lam, t = (np.asarray(a, dtype=float).copy() for a in sol)
    src = QpSolution(lay, y.copy(), pi.copy(), lam.copy(), t.copy())
    g = QpSolution(lay, y, pi, lam, t)
    for n in range(N - 1):
        g.x(n)[:] = src.x(n + 1)
        if g.u(n).shape == src.u(n + 1).shape:
            g.u(n)[:] = src.u(n + 1)
        g.pi_stage(n)[:] = src.pi_stage(n + 1)
        if g.lam_stage(n).shape == src.lam_stage(n + 1).shape:
            g.lam_stage(n)[:] = src.lam_stage(n + 1)
            g.t_stage(n)[:] = src.t_stage(n + 1)
    g.x(N - 1)[:] = src.x(N)
    A = batch.stage_view("A", N - 1)[0]
    Bm = batch.stage_view("B", N - 1)[0]
    b = batch.stage_view("b", N - 1)[0] if "b" in batch.fields else np.zeros(d.nx[N])
    g.x(N)[:] = A @ g.x(N - 1) + Bm @ g.u(N - 1) + b
    nu0 = int(d.nu[0])
    m0 = int(d.nb[0]) + int(d.ng[0])
    xrows = [(i, int(k) - nu0) for i, k in enumerate(batch.idxb[0]) if int(k) >= nu0]
    if xrows:
        lam0 = g.lam_stage(0)
        t0 = g.t_stage(0)
        for i, _ in xrows:
            lam0[i] = 0.0
            lam0[m0 + i] = 0.0
        r = orc.residuals(batch, g.y[None], g.pi[None], g.lam[None], g.t[None])
        gap = r["r_g"][0][lay.x_off[0]: lay.x_off[0] + int(d.nx[0])]
        for i, c in xrows:
            if gap[c] >= 0.0:
                lam0[i] = gap[c]
            else:
                lam0[m0 + i] = -gap[c]
            t0[i] = 0.0
            t0[m0 + i] = 0.0
    return g.y, g.pi, g.lam, g.t


def run_closed_loop(cfg, steps, arg, warm_start="primal_dual", compare_cold=False):
    """Returns dict(states, inputs, iters, cold_iters, status)."""
    from paper_2003_02547_b200 import OcpQpBatch
    from paper_2003_02547_b200.mpc import default_x0, gen_mass_spring, mass_spring_dynamics

    M = cfg.masses
    A, Bm = mass_spring_dynamics(M, cfg.ts)
    x = np.asarray(cfg.x0, dtype=float) if cfg.x0 is not None else default_x0(M)
    states, inputs, iters, cold, status = [x.copy()], [], [], [], []
    guess = None
    for _ in range(steps):
        batch = OcpQpBatch.from_qps([gen_mass_spring(replace(cfg, x0=x))])
        a = replace(arg, warm_start=warm_start if guess is not None else "none")
        out = orc.solve(batch, a, nthreads=1, trace=False,
                        guess=None if guess is None else tuple(v[None] for v in guess))
        iters.append(int(out["iters"][0]))
        status.append(int(out["status"][0]))
        if compare_cold:
            c = orc.solve(batch, replace(arg, warm_start="none"), nthreads=1, trace=False)
            cold.append(int(c["iters"][0]))
        u0 = out["y"][0][batch.layout.u_off[0]: batch.layout.u_off[0] + M - 1].copy()
        inputs.append(u0)
        x = A @ x + Bm @ u0
        states.append(x.copy())
        guess = shift_guess(batch, (out["y"][0], out["pi"][0], out["lam"][0], out["t"][0]))
    return dict(states=np.array(states), inputs=np.array(inputs), iters=np.array(iters),
                cold_iters=np.array(cold), status=np.array(status))
