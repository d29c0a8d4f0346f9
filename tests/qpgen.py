"""Random feasible OCP-QP instances for tests (shared by the golden script).

Builds problems as plain field dictionaries so the same instance can populate
either this package's ``OcpQp`` or the reference's (for golden generation).
Feasible by construction: a trajectory (u, x) is rolled out first and every
bound is placed around it.  Exercises box subsets, general rows, soft rows,
per-side masks, infinite (inactive) sides and an equality-fixed x0.
"""

from __future__ import annotations

import numpy as np


def random_ocp_fields(seed, N=5, nx=4, nu=2, nb=3, ng=1, ns=1, fix_x0=False,
                      mask_last=True, inf_side=True, decay=0.5):
    """Return (dims, stages, dyn): dims = dict(N, nx, nu, nb, ng, ns lists)."""
    rng = np.random.default_rng(seed)
    nxl = [nx] * (N + 1)
    nul = [nu] * N + [0]
    nbl = []
    for n in range(N + 1):
        if fix_x0 and n == 0:
            nbl.append(nul[0] + nx)
        else:
            nbl.append(min(nb, nul[n] + nx))
    ngl = [ng] * (N + 1)
    nsl = [min(ns, nbl[n] + ngl[n]) for n in range(N + 1)]
    if fix_x0:
        nsl[0] = min(ns, nul[0] + ngl[0])
    u_tr = [rng.uniform(-1.0, 1.0, nul[n]) for n in range(N + 1)]
    x_tr = [rng.uniform(-1.0, 1.0, nx)]
    dyn = []
    for n in range(N):
        A = decay * rng.standard_normal((nx, nx))
        B = rng.standard_normal((nx, nul[n]))
        b = rng.uniform(-0.2, 0.2, nx)
        dyn.append(dict(A=A, B=B, b=b))
        x_tr.append(A @ x_tr[n] + B @ u_tr[n] + b)
    stages = []
    for n in range(N + 1):
        nw = nul[n] + nx
        F = rng.standard_normal((nw, nw))
        H = F @ F.T + np.eye(nw)
        H = 0.5 * (H + H.T)
        st = dict(R=H[:nul[n], :nul[n]].copy(), S=H[:nul[n], nul[n]:].copy(),
                  Q=H[nul[n]:, nul[n]:].copy(),
                  r=0.3 * rng.standard_normal(nul[n]), q=0.3 * rng.standard_normal(nx))
        w = np.concatenate([u_tr[n], x_tr[n]])
        if fix_x0 and n == 0:
            idxb = np.arange(nw)
            lb = np.concatenate([u_tr[0] - 2.0, x_tr[0]])
            ub = np.concatenate([u_tr[0] + 2.0, x_tr[0]])
        else:
            idxb = np.sort(rng.choice(nw, nbl[n], replace=False))
            lb = w[idxb] - rng.uniform(0.5, 2.0, nbl[n])
            ub = w[idxb] + rng.uniform(0.5, 2.0, nbl[n])
        if inf_side and nbl[n] >= 2 and not (fix_x0 and n == 0):
            ub[-1] = np.inf       # one-sided box row: upper side inactive
        st.update(idxb=idxb, lb=lb, ub=ub)
        if ngl[n]:
            C = rng.standard_normal((ngl[n], nx))
            D = rng.standard_normal((ngl[n], nul[n]))
            cw = D @ u_tr[n] + C @ x_tr[n]
            st.update(C=C, D=D, lg=cw - rng.uniform(0.5, 2.0, ngl[n]),
                      ug=cw + rng.uniform(0.5, 2.0, ngl[n]))
        if nsl[n]:
            if fix_x0 and n == 0:
                pool = np.concatenate([np.arange(nul[0]), nbl[0] + np.arange(ngl[0])])
            else:
                pool = np.arange(nbl[n] + ngl[n])
            idxs = np.sort(rng.choice(pool, nsl[n], replace=False))
            st.update(idxs=idxs, Zl=rng.uniform(0.5, 2.0, nsl[n]), Zu=rng.uniform(0.5, 2.0, nsl[n]),
                      zl=rng.uniform(0.0, 0.3, nsl[n]), zu=rng.uniform(0.0, 0.3, nsl[n]))
        if mask_last and nbl[n] + ngl[n] and not (fix_x0 and n == 0):
            maskl = np.ones(nbl[n] + ngl[n])
            maskl[-1] = 0.0
            st["maskl"] = maskl
        stages.append(st)
    dims = dict(N=N, nx=nxl, nu=nul, nb=nbl, ng=ngl, ns=nsl)
    return dims, stages, dyn


def build_qp(module, dims, stages, dyn):
    """Populate ``module.OcpQp`` (this package or the reference) from fields."""
    qp = module.OcpQp(module.OcpQpDim(dims["N"], dims["nx"], dims["nu"], dims["nb"],
                                      dims["ng"], dims["ns"]))
    order = ["idxb", "idxs"]
    for n, st in enumerate(stages):
        for name in order:
            if name in st:
                qp.set_field(name, n, st[name])
        for name, val in st.items():
            if name not in order:
                qp.set_field(name, n, val)
    for n, dd in enumerate(dyn):
        for name, val in dd.items():
            qp.set_field(name, n, val)
    return qp


def scalar_lqr(module, bounds=False):
    """1-state / 1-input LQR with unit weights (the reference's hand example)."""
    if bounds:
        qp = module.OcpQp(module.OcpQpDim(1, nx=[1, 1], nu=[1, 0], nb=[2, 1]))
        qp.set_field("idxb", 0, [0, 1])
        qp.set_field("lb", 0, [-50.0, 3.0])
        qp.set_field("ub", 0, [50.0, 3.0])
        qp.set_field("idxb", 1, [0])
        qp.set_field("lb", 1, [-50.0])
        qp.set_field("ub", 1, [50.0])
    else:
        qp = module.OcpQp(module.OcpQpDim(1, nx=[1, 1], nu=[1, 0]))
    qp.set_field("Q", 0, [[1.0]])
    qp.set_field("R", 0, [[1.0]])
    qp.set_field("Q", 1, [[1.0]])
    qp.set_field("A", 0, [[1.0]])
    qp.set_field("B", 0, [[1.0]])
    return qp


def rank_deficient(module):
    """Two-state QP whose terminal stage Hessian diag(1, 1e-34) is positive
    definite (Cholesky succeeds) but numerically rank deficient for the QR
    array algorithm (linalg.py:176-184): robust mode raises RankDeficient."""
    qp = module.OcpQp(module.OcpQpDim(1, nx=[2, 2], nu=[1, 0], nb=[1, 0]))
    qp.set_field("idxb", 0, [0])
    qp.set_field("lb", 0, [-1.0])
    qp.set_field("ub", 0, [1.0])
    qp.set_field("Q", 0, [[1.0, 0.0], [0.0, 1e-34]])
    qp.set_field("R", 0, [[1.0]])
    qp.set_field("q", 0, [1.0, 0.0])
    qp.set_field("Q", 1, [[1.0, 0.0], [0.0, 1e-34]])
    qp.set_field("A", 0, [[1.0, 0.0], [0.0, 1.0]])
    qp.set_field("B", 0, [[1.0], [0.0]])
    return qp
