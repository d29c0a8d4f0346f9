"""Seeded synthetic inputs for the five BASELINE configurations.

There is no public dataset for this path; every config is a
seeded generator with the shapes and value distributions BASELINE.json names.
One RNG per QP, ``np.random.default_rng(SeedSequence([cfg, i]))``, with the
draw order fixed below, so a QP is reproducible from (cfg, i) alone and the
same arrays feed the packed GPU batch and the reference ``OcpQp`` objects.

* cfg 0/1: 4-mass spring chain (nx=8, nu=3, actuators on masses 1-3), exact
  discretisation ``expm([[Ac, Bc], [0, 0]] Ts)`` with Ts=0.5 as in
  mass_spring.py:99-114, N=15, Q=I, R=2I, |u|<=0.5, |x|<=4, x0 positions
  U(-1,1), velocities 0, imposed by lbx=ubx=x0 (mass_spring.py:147-148).
* cfg 2: 12-mass chain, actuators on masses 1,4,7,10 (nu=4), N=30, Q=I, R=I,
  |u|<=1, |x|<=4, x0 positions U(-1.5,1.5).
* cfg 3: random stage-varying nx=30, nu=10, N=50, ng=10:
  A_k = (I + 0.1 G)/rho(I + 0.1 G), B_k ~ N(0,1), b_k ~ N(0, 0.1^2),
  Q_k = M M'/nx + 1e-2 I, R_k = L L'/nu + 1e-2 I, q, r ~ N(0,1),
  |u|<=1, |x|<=5, general rows C x + D u <= d with lg = -inf,
  d = 1 + |N(0,1)|, C, D Gaussian scaled by 0.1 (documented deviation: the
  literal scaling is infeasible for the reference oracle), terminal stage C
  only; x0 ~ N(0,1).
* cfg 4: the cfg-3 generator with nx=60, nu=20, N=100 and ng=0.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .batch import OcpQpBatch
from .qp_data import OcpQpDim

__all__ = ["CONFIGS", "ConfigSpec", "chain_dynamics", "make_batch", "make_qps",
           "config_dim"]


@dataclass(frozen=True)
class ConfigSpec:
    cfg: int
    kind: str            # "chain" | "random"
    batch: int
    N: int
    nx: int
    nu: int
    ng: int = 0
    masses: int = 0
    actuators: tuple = ()
    r_weight: float = 1.0
    u_bound: float = 1.0
    x_bound: float = 4.0
    x0_range: float = 1.0
    cd_scale: float = 0.1


CONFIGS = {
    0: ConfigSpec(0, "chain", 1, 15, 8, 3, masses=4, actuators=(0, 1, 2), r_weight=2.0,
                  u_bound=0.5, x_bound=4.0, x0_range=1.0),
    1: ConfigSpec(1, "chain", 1024, 15, 8, 3, masses=4, actuators=(0, 1, 2), r_weight=2.0,
                  u_bound=0.5, x_bound=4.0, x0_range=1.0),
    2: ConfigSpec(2, "chain", 8192, 30, 24, 4, masses=12, actuators=(0, 3, 6, 9),
                  r_weight=1.0, u_bound=1.0, x_bound=4.0, x0_range=1.5),
    3: ConfigSpec(3, "random", 512, 50, 30, 10, ng=10, u_bound=1.0, x_bound=5.0),
    4: ConfigSpec(4, "random", 256, 100, 60, 20, ng=0, u_bound=1.0, x_bound=5.0),
}


def chain_dynamics(masses, ts, actuators):
    """Exactly discretised (A, B) of a spring chain (mass_spring.py:99-114)."""
    import scipy.linalg

    M = masses
    T = -2.0 * np.eye(M) + np.eye(M, k=1) + np.eye(M, k=-1)
    nx, nu = 2 * M, len(actuators)
    Ac = np.zeros((nx, nx))
    Ac[:M, M:] = np.eye(M)
    Ac[M:, :M] = T
    Bc = np.zeros((nx, nu))
    Bc[M:, :] = np.eye(M)[:, list(actuators)]
    aug = np.zeros((nx + nu, nx + nu))
    aug[:nx, :nx] = Ac
    aug[:nx, nx:] = Bc
    E = scipy.linalg.expm(aug * ts)
    return E[:nx, :nx], E[:nx, nx:]


def config_dim(spec: ConfigSpec, N=None) -> OcpQpDim:
    N = spec.N if N is None else N
    nx, nu = spec.nx, spec.nu
    return OcpQpDim(N, nx=[nx] * (N + 1), nu=[nu] * N + [0],
                    nb=[nu + nx] * N + [nx], ng=[spec.ng] * (N + 1), ns=[0] * (N + 1))


def _rng(cfg, i):
    return np.random.default_rng(np.random.SeedSequence([cfg, i]))


def _chain_x0(spec, i):
    rng = _rng(spec.cfg, i)
    M = spec.masses
    x0 = np.zeros(2 * M)
    x0[:M] = rng.uniform(-spec.x0_range, spec.x0_range, M)
    return x0


def _random_draws(spec, i, N):
    """Per-QP arrays of the random generator, blocked draw order (see module doc)."""
    rng = _rng(spec.cfg, i)
    nx, nu, ng = spec.nx, spec.nu, spec.ng
    G = rng.standard_normal((N, nx, nx))
    A = np.eye(nx)[None] + 0.1 * G
    rho = np.max(np.abs(np.linalg.eigvals(A)), axis=1)
    A = A / rho[:, None, None]
    B = rng.standard_normal((N, nx, nu))
    b = 0.1 * rng.standard_normal((N, nx))
    Mq = rng.standard_normal((N + 1, nx, nx))
    Q = Mq @ np.swapaxes(Mq, 1, 2) / nx + 1e-2 * np.eye(nx)[None]
    Q = 0.5 * (Q + np.swapaxes(Q, 1, 2))
    q = rng.standard_normal((N + 1, nx))
    Lr = rng.standard_normal((N, nu, nu))
    R = Lr @ np.swapaxes(Lr, 1, 2) / nu + 1e-2 * np.eye(nu)[None]
    R = 0.5 * (R + np.swapaxes(R, 1, 2))
    r = rng.standard_normal((N, nu))
    C = spec.cd_scale * rng.standard_normal((N + 1, ng, nx))
    D = spec.cd_scale * rng.standard_normal((N, ng, nu))
    dg = 1.0 + np.abs(rng.standard_normal((N + 1, ng)))
    x0 = rng.standard_normal(nx)
    return dict(A=A, B=B, b=b, Q=Q, q=q, R=R, r=r, C=C, D=D, dg=dg, x0=x0)


def make_batch(cfg, batch=None, start=0, N=None) -> OcpQpBatch:
    """Packed batch of config ``cfg`` for QP indices start..start+batch-1."""
    spec = CONFIGS[cfg]
    B = spec.batch if batch is None else int(batch)
    N = spec.N if N is None else int(N)
    dim = config_dim(spec, N)
    nx, nu = spec.nx, spec.nu
    out = OcpQpBatch(dim, B)
    if spec.kind == "chain":
        A, Bm = chain_dynamics(spec.masses, 0.5, spec.actuators)
        for name, per_qp in (("A", False), ("B", False), ("Q", False), ("R", False),
                             ("lb", True), ("ub", True)):
            out.alloc(name, per_qp, 0.0)
        for n in range(N + 1):
            out.stage_view("Q", n)[:] = np.eye(nx)
            if n < N:
                out.stage_view("A", n)[:] = A
                out.stage_view("B", n)[:] = Bm
                out.stage_view("R", n)[:] = spec.r_weight * np.eye(nu)
                lb = np.concatenate([-spec.u_bound * np.ones(nu), -spec.x_bound * np.ones(nx)])
            else:
                lb = -spec.x_bound * np.ones(nx)
            out.stage_view("lb", n)[:] = lb
            out.stage_view("ub", n)[:] = -lb
        lb0 = out.stage_view("lb", 0)
        ub0 = out.stage_view("ub", 0)
        for k in range(B):
            x0 = _chain_x0(spec, start + k)
            lb0[k, nu:] = x0
            ub0[k, nu:] = x0
        return out
    # random stage-varying configs: everything per QP
    for name in ("A", "B", "b", "Q", "R", "q", "r", "lb", "ub"):
        out.alloc(name, True, 0.0)
    if spec.ng:
        for name in ("C", "D", "lg", "ug"):
            out.alloc(name, True, 0.0)
    # per-QP draws are independent (one RNG per QP); LAPACK eigvals releases
    # the GIL, so a thread pool generates them in parallel, bit-identically
    from concurrent.futures import ThreadPoolExecutor
    import os

    workers = max(1, min(B, os.cpu_count() or 1, 32))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        draws = list(ex.map(lambda k: _random_draws(spec, start + k, N), range(B)))
    for k in range(B):
        dr = draws[k]
        draws[k] = None
        f = out.fields
        f["A"][k] = dr["A"].reshape(-1)
        f["B"][k] = dr["B"].reshape(-1)
        f["b"][k] = dr["b"].reshape(-1)
        f["Q"][k] = dr["Q"].reshape(-1)
        f["q"][k] = dr["q"].reshape(-1)
        f["R"][k] = dr["R"].reshape(-1)
        f["r"][k] = dr["r"].reshape(-1)
        lbs, ubs = [], []
        for n in range(N + 1):
            if n < N:
                lb = np.concatenate([-spec.u_bound * np.ones(nu), -spec.x_bound * np.ones(nx)])
            else:
                lb = -spec.x_bound * np.ones(nx)
            ub = -lb
            if n == 0:
                lb[nu:] = dr["x0"]
                ub[nu:] = dr["x0"]
            lbs.append(lb)
            ubs.append(ub)
        f["lb"][k] = np.concatenate(lbs)
        f["ub"][k] = np.concatenate(ubs)
        if spec.ng:
            f["C"][k] = dr["C"].reshape(-1)
            f["D"][k] = dr["D"].reshape(-1)
            f["lg"][k] = -np.inf
            f["ug"][k] = dr["dg"].reshape(-1)
    return out


def make_qps(cfg, indices, N=None):
    """Reference-style OcpQp objects for the given QP indices (drop-in path)."""
    out = []
    for i in indices:
        bi = make_batch(cfg, batch=1, start=int(i), N=N)
        out.append(bi.qp(0))
    return out
