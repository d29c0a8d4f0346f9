"""Generate golden vectors from the REAL reference package (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (/root/reference/pkg/src/mpcqp, pure Python) is imported here
only; it does not exist on the GPU box, so tests read the committed .npz
fixtures written by this script.  Inputs are NOT stored for the seeded
generators -- they are regenerated bit-identically from
paper_2003_02547_b200.generators (BASELINE configs) and tests/qpgen.py
(random feasible instances) with the recorded parameters; only the
reference's outputs are stored.

Fixtures:
  solve_cfg.npz      speed-mode solves (tol 1e-8) of the first QPs of configs 0-4
  solve_random.npz   speed-mode solves of random instances with soft rows,
                     masks, one-sided rows, general rows, fixed x0
  newton.npz         riccati_factor + solve Newton steps at random iterates,
                     with the cost-to-go matrices P[n] and gains K[n]
  residuals.npz      compute_residuals at random points
  known.npz          hand-derivable answers (scalar LQR) and failure statuses
  modes.npz          balance / robust / square-root / speed_abs solves (MODES),
                     their Failure ladders and the robust-mode RankDeficient raise
  pcond_full.npz     config 4 (N = 100) partial condensing -> solve -> expand
  dense_eq.npz       dense QPs with equality constraints (Schur / null-space)
  closed_loop.npz    run_closed_loop trajectories / iteration counts (warm and
                     cold) and one _shift_guess
  qp_files/          qp_write text files and `mpcqp solve` CLI reports
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import mpcqp  # noqa: E402  (the reference)
import mpcqp.kkt_ocp as ko  # noqa: E402
from mpcqp.view import QpSolution as RefSol, make_view  # noqa: E402

import qpgen  # noqa: E402
from paper_2003_02547_b200.generators import make_batch  # noqa: E402

STATUS = {"Success": 0, "MaxIter": 1, "MinStep": 2, "NaNDetected": 3, "Failure": 4}
ARG = mpcqp.mode_preset("speed").with_tol(1e-8)

# (cfg, indices, N) of the config fixtures
CFG_CASES = [(0, [0], None), (1, list(range(12)), None), (2, [0, 1, 2], None),
             (3, [0, 1, 2], None), (4, [0], None)]
# random instances: (seed, kwargs)
RANDOM_CASES = [
    (11, dict(N=5, nx=4, nu=2, nb=3, ng=1, ns=1)),
    (12, dict(N=6, nx=3, nu=2, nb=4, ng=2, ns=2, fix_x0=True)),
    (13, dict(N=4, nx=5, nu=1, nb=2, ng=0, ns=0)),
    (14, dict(N=7, nx=4, nu=3, nb=5, ng=2, ns=0, mask_last=False, inf_side=False)),
    (15, dict(N=3, nx=2, nu=2, nb=4, ng=1, ns=3, fix_x0=True)),
    (16, dict(N=8, nx=6, nu=2, nb=8, ng=0, ns=2)),
]


def to_ref(qp_local):
    """Copy a package OcpQp into a reference OcpQp (same field catalog)."""
    d = qp_local.dim
    ref = mpcqp.OcpQp(mpcqp.OcpQpDim(d.N, d.nx, d.nu, d.nb, d.ng, d.ns))
    for n in range(d.N + 1):
        for k, v in qp_local._stages[n].items():
            ref._stages[n][k] = np.array(v, copy=True)
    for n in range(d.N):
        for k, v in qp_local._dyn[n].items():
            ref._dyn[n][k] = np.array(v, copy=True)
    ref._rev += 1
    return ref


def pack_report(rep):
    s = rep.solution
    st = rep.stats
    tr = np.array([[r.alpha_aff, r.alpha, r.mu, r.sigma, r.res_g, r.res_b, r.res_d, r.res_m]
                   for r in st.trace]).reshape(-1, 8)
    return dict(status=STATUS[st.status.value], iters=st.iterations, y=s.y, pi=s.pi, lam=s.lam,
                t=s.t, res=np.array([st.res_g, st.res_b, st.res_d, st.res_m, st.mu]),
                flops=st.flops, trace=tr)


def solve_cfg():
    out = {}
    for cfg, idx, N in CFG_CASES:
        for i in idx:
            qp = to_ref(make_batch(cfg, batch=1, start=i, N=N).qp(0))
            rep = mpcqp.solve_ocp_qp(qp, ARG)
            for k, v in pack_report(rep).items():
                out[f"c{cfg}_q{i}_{k}"] = v
            print("cfg", cfg, "qp", i, rep.status.value, rep.iterations, flush=True)
    out["cases"] = np.array([[c, i] for c, idx, _ in CFG_CASES for i in idx])
    np.savez_compressed(HERE / "solve_cfg.npz", **out)


def solve_random():
    out = {}
    for seed, kw in RANDOM_CASES:
        qp = qpgen.build_qp(mpcqp, *qpgen.random_ocp_fields(seed, **kw))
        rep = mpcqp.solve_ocp_qp(qp, ARG)
        for k, v in pack_report(rep).items():
            out[f"s{seed}_{k}"] = v
        print("random", seed, rep.status.value, rep.iterations, flush=True)
    np.savez_compressed(HERE / "solve_random.npz", **out)


def random_iterate(rng, vw, spread=(0.1, 5.0)):
    it = RefSol(vw)
    it.y[:] = rng.standard_normal(vw.ny)
    it.pi[:] = rng.standard_normal(vw.ne)
    it.lam[:] = np.where(vw.act, rng.uniform(*spread, vw.nc), 0.0)
    it.t[:] = np.where(vw.act, rng.uniform(*spread, vw.nc), 0.0)
    return it


def newton():
    out = {}
    rng = np.random.default_rng(2024)
    for seed, kw in RANDOM_CASES:
        qp = qpgen.build_qp(mpcqp, *qpgen.random_ocp_fields(seed, **kw))
        vw = make_view(qp)
        it = random_iterate(rng, vw)
        res = mpcqp.compute_residuals(qp, it)
        rm = np.where(vw.act, it.lam * it.t, 0.0)
        fac = ko.riccati_factor(qp, it)
        step = fac.solve(res.r_g, res.r_b, res.r_d, rm)
        P = np.concatenate([fac.p_matrix(n).reshape(-1) for n in range(qp.dim.N + 1)])
        K = np.concatenate([fac.K[n].reshape(-1) for n in range(qp.dim.N + 1)])
        for k, v in dict(y=it.y, pi=it.pi, lam=it.lam, t=it.t, r_g=res.r_g, r_b=res.r_b,
                         r_d=res.r_d, r_m=rm, dy=step.y, dpi=step.pi, dlam=step.lam,
                         dt=step.t, P=P, K=K).items():
            out[f"s{seed}_{k}"] = v
    # the same at BASELINE config shapes
    for cfg in (1, 2, 3):
        qp = to_ref(make_batch(cfg, batch=1, start=7).qp(0))
        vw = make_view(qp)
        it = random_iterate(rng, vw)
        res = mpcqp.compute_residuals(qp, it)
        rm = np.where(vw.act, it.lam * it.t, 0.0)
        fac = ko.riccati_factor(qp, it)
        step = fac.solve(res.r_g, res.r_b, res.r_d, rm)
        for k, v in dict(y=it.y, pi=it.pi, lam=it.lam, t=it.t, r_g=res.r_g, r_b=res.r_b,
                         r_d=res.r_d, r_m=rm, dy=step.y, dpi=step.pi, dlam=step.lam,
                         dt=step.t).items():
            out[f"c{cfg}_{k}"] = v
    np.savez_compressed(HERE / "newton.npz", **out)


def residuals():
    out = {}
    rng = np.random.default_rng(77)
    for seed, kw in RANDOM_CASES:
        qp = qpgen.build_qp(mpcqp, *qpgen.random_ocp_fields(seed, **kw))
        vw = make_view(qp)
        it = random_iterate(rng, vw)
        r = mpcqp.compute_residuals(qp, it)
        for k, v in dict(y=it.y, pi=it.pi, lam=it.lam, t=it.t, r_g=r.r_g, r_b=r.r_b, r_d=r.r_d,
                         r_m=r.r_m, norms=np.array([r.res_g, r.res_b, r.res_d, r.res_m, r.mu])).items():
            out[f"s{seed}_{k}"] = v
    np.savez_compressed(HERE / "residuals.npz", **out)


def known():
    out = {}
    qp = qpgen.scalar_lqr(mpcqp)
    fac = ko.riccati_factor(qp, RefSol(make_view(qp)))
    out["lqr_P1"] = fac.p_matrix(1)[0, 0]
    out["lqr_K0"] = fac.K[0][0, 0]
    out["lqr_P0"] = fac.p_matrix(0)[0, 0]
    rep = mpcqp.solve_ocp_qp(qpgen.scalar_lqr(mpcqp, bounds=True), ARG)
    out["lqr_bounds_u0"] = rep.solution.u(0)[0]
    out["lqr_bounds_status"] = STATUS[rep.status.value]
    # indefinite input weight: Failure after the regularised retry
    q = qpgen.scalar_lqr(mpcqp)
    q.set_field("r", 0, [1.0])
    q.set_field("R", 0, [[-1.0]])
    q.set_field("Q", 0, [[-1.0]])
    q.set_field("Q", 1, [[-1.0]])
    rep = mpcqp.solve_ocp_qp(q, ARG)
    out["indef_status"] = STATUS[rep.status.value]
    out["indef_iters"] = rep.iterations
    out["indef_flops"] = rep.stats.flops
    # crossed bounds: never Success
    q = qpgen.scalar_lqr(mpcqp, bounds=True)
    q.set_field("lb", 1, [1.0])
    q.set_field("ub", 1, [0.0])
    rep = mpcqp.solve_ocp_qp(q, ARG)
    out["infeas_status"] = STATUS[rep.status.value]
    out["infeas_iters"] = rep.iterations
    np.savez_compressed(HERE / "known.npz", **out)
    print({k: float(v) for k, v in out.items()})


# partial condensing cases: (name, source, N1) -- source is a RANDOM_CASES-style
# (seed, kwargs) without soft rows, or ("cfg", cfg, N) for a BASELINE generator
PCOND_CASES = [
    ("r21", (21, dict(N=8, nx=3, nu=2, nb=4, ng=1, ns=0, fix_x0=True)), 4),
    ("r22", (22, dict(N=7, nx=2, nu=1, nb=3, ng=0, ns=0, fix_x0=True)), 3),
    ("r23", (23, dict(N=6, nx=3, nu=2, nb=5, ng=2, ns=0, fix_x0=True)), 1),
    ("r24", (24, dict(N=5, nx=4, nu=2, nb=6, ng=1, ns=0, fix_x0=True, mask_last=False)), 5),
    ("c4", ("cfg", 4, 10), 5),
    ("c1", ("cfg", 1, None), 5),
]
PCOND_FIELDS = ("Q", "S", "R", "q", "r", "idxb", "lb", "ub", "C", "D", "lg", "ug", "maskl", "masku")


def pcond_source(src):
    if src[0] == "cfg":
        _, cfg, N = src
        return to_ref(make_batch(cfg, batch=1, start=0, N=N).qp(0))
    seed, kw = src
    return qpgen.build_qp(mpcqp, *qpgen.random_ocp_fields(seed, **kw))


def pcond():
    out = {}
    for name, src, N1 in PCOND_CASES:
        qp = pcond_source(src)
        qp2, pmap = mpcqp.partial_condense(qp, N1)
        d2 = qp2.dim
        out[f"{name}_dims"] = np.array([d2.nx, d2.nu, d2.nb, d2.ng])
        for n in range(d2.N + 1):
            for f in PCOND_FIELDS:
                out[f"{name}_s{n}_{f}"] = qp2.get_field(f, n)
            if n < d2.N:
                for f in ("A", "B", "b"):
                    out[f"{name}_s{n}_{f}"] = qp2.get_field(f, n)
        rep = mpcqp.solve_ocp_qp(qp2, ARG)
        full = mpcqp.partial_expand(rep.solution, pmap, qp)
        for k, v in pack_report(rep).items():
            out[f"{name}_short_{k}"] = v
        for k in ("y", "pi", "lam", "t"):
            out[f"{name}_full_{k}"] = getattr(full, k)
        direct = mpcqp.solve_ocp_qp(qp, ARG)
        out[f"{name}_direct_iters"] = direct.iterations
        out[f"{name}_direct_y"] = direct.solution.y
        print("pcond", name, d2.N, rep.status.value, rep.iterations, direct.iterations, flush=True)
    np.savez_compressed(HERE / "pcond.npz", **out)


# BASELINE config 4's second way at full size: N = 100 -> N2 = 20 blocks of 5
PCOND_FULL_QPS = [0, 1, 2]


def pcond_full():
    """Reference partial_condense(qp, 5) -> solve -> partial_expand on full-size
    config-4 QPs (N = 100, nx = 60, nu = 20): condensed-solve status /
    iterations / final norms and the expanded solution (the condensed fields
    themselves are 11 MB per QP; their restatement is pinned by pcond.npz)."""
    out = {}
    for i in PCOND_FULL_QPS:
        qp = to_ref(make_batch(4, batch=1, start=i).qp(0))
        qp2, pmap = mpcqp.partial_condense(qp, 5)
        rep = mpcqp.solve_ocp_qp(qp2, ARG)
        full = mpcqp.partial_expand(rep.solution, pmap, qp)
        r = pack_report(rep)
        for k in ("status", "iters", "res", "flops"):
            out[f"q{i}_short_{k}"] = r[k]
        for k in ("y", "pi", "lam", "t"):
            out[f"q{i}_full_{k}"] = getattr(full, k)
        print("pcond_full", i, rep.status.value, rep.iterations, flush=True)
    out["qps"] = np.array(PCOND_FULL_QPS)
    np.savez_compressed(HERE / "pcond_full.npz", **out)


# full condensing (condensing.py:160-429) + the dense-QP IPM (solver.py:98-100)
FCOND_CASES = [
    ("f21", (21, dict(N=8, nx=3, nu=2, nb=4, ng=1, ns=0, fix_x0=True)), None),
    ("f23", (23, dict(N=6, nx=3, nu=2, nb=5, ng=2, ns=0, fix_x0=True)), None),
    ("f25", (25, dict(N=5, nx=3, nu=2, nb=3, ng=1, ns=0, fix_x0=False)), None),
    ("f26", (26, dict(N=4, nx=4, nu=1, nb=4, ng=0, ns=0, fix_x0=False, mask_last=False)), None),
    ("f27", (27, dict(N=6, nx=3, nu=2, nb=5, ng=1, ns=0, fix_x0=True)), True),
    ("c1", ("cfg", 1, None), None),
    ("c2", ("cfg", 2, 10), None),
]
FCOND_FIELDS = ("H", "g", "idxb", "lb", "ub", "C", "lg", "ug", "maskl", "masku")


def fcond():
    out = {}
    for name, src, keep in FCOND_CASES:
        qp = pcond_source(src)
        dq, cmap = mpcqp.condense(qp, keep_x0=keep)
        out[f"{name}_dims"] = np.array([dq.nv, dq.ne, dq.nb, dq.ng, dq.ns, int(cmap.keep_x0)])
        for f in FCOND_FIELDS:
            out[f"{name}_{f}"] = dq.get_field(f)
        rep = mpcqp.solve_dense_qp(dq, ARG)
        for k, v in pack_report(rep).items():
            out[f"{name}_dense_{k}"] = v
        full = mpcqp.expand_solution(rep.solution, cmap, qp)
        for k in ("y", "pi", "lam", "t"):
            out[f"{name}_full_{k}"] = getattr(full, k)
        direct = mpcqp.solve_ocp_qp(qp, ARG)
        out[f"{name}_direct_iters"] = direct.iterations
        out[f"{name}_direct_y"] = direct.solution.y
        print("fcond", name, dq.nv, dq.ng, cmap.keep_x0, rep.status.value, rep.iterations,
              direct.iterations, flush=True)
    np.savez_compressed(HERE / "fcond.npz", **out)


def fcond_sqrt():
    """condense(variant="square_root") (condensing.py:134-146) of the fcond cases: the
    Hessian and gradient of the dense QP (every other field does not depend on the
    cost recursion), and the NotPositiveDefinite raise on a semidefinite stage cost."""
    out = {}
    for name, src, keep in FCOND_CASES:
        qp = pcond_source(src)
        dq, cmap = mpcqp.condense(qp, keep_x0=keep, variant="square_root")
        dc, _ = mpcqp.condense(qp, keep_x0=keep)
        out[f"{name}_H"] = dq.get_field("H")
        out[f"{name}_g"] = dq.get_field("g")
        out[f"{name}_H_vs_classical"] = np.max(np.abs(dq.get_field("H") - dc.get_field("H")))
        print("fcond_sqrt", name, dq.nv, out[f"{name}_H_vs_classical"], flush=True)
    qp = pcond_source(FCOND_CASES[0][1])
    qp.set_field("Q", 2, np.zeros((3, 3)))
    try:
        mpcqp.condense(qp, variant="square_root")
        out["npd_raises"] = np.array(0)
    except mpcqp.errors.NotPositiveDefinite:
        out["npd_raises"] = np.array(1)
    print("fcond_sqrt npd", int(out["npd_raises"]), flush=True)
    np.savez_compressed(HERE / "fcond_sqrt.npz", **out)


# condensing with soft rows (condensing.py:289-334, 523-534, 592-601)
SOFT_CASES = [
    ("s31", (31, dict(N=5, nx=3, nu=2, nb=4, ng=1, ns=2, fix_x0=True)), None, 2),
    ("s32", (32, dict(N=4, nx=3, nu=2, nb=3, ng=2, ns=2)), None, 3),
    ("s33", (33, dict(N=6, nx=2, nu=2, nb=4, ng=1, ns=3, fix_x0=True)), True, 4),
    ("s34", (34, dict(N=5, nx=4, nu=1, nb=5, ng=0, ns=2, mask_last=False)), None, 2),
]
SOFT_DFIELDS = FCOND_FIELDS + ("idxs", "Zl", "Zu", "zl", "zu", "sl_lb", "su_lb")
SOFT_PFIELDS = PCOND_FIELDS + ("idxs", "Zl", "Zu", "zl", "zu", "sl_lb", "su_lb")


def soft_cond():
    out = {}
    for name, src, keep, N1 in SOFT_CASES:
        qp = pcond_source(src)
        dq, cmap = mpcqp.condense(qp, keep_x0=keep)
        out[f"{name}_dims"] = np.array([dq.nv, dq.ne, dq.nb, dq.ng, dq.ns, int(cmap.keep_x0)])
        for f in SOFT_DFIELDS:
            out[f"{name}_{f}"] = dq.get_field(f)
        rep = mpcqp.solve_dense_qp(dq, ARG)
        for k, v in pack_report(rep).items():
            out[f"{name}_dense_{k}"] = v
        full = mpcqp.expand_solution(rep.solution, cmap, qp)
        for k in ("y", "pi", "lam", "t"):
            out[f"{name}_full_{k}"] = getattr(full, k)
        qp2, pmap = mpcqp.partial_condense(qp, N1)
        d2 = qp2.dim
        out[f"{name}_p_dims"] = np.array([d2.nx, d2.nu, d2.nb, d2.ng, d2.ns])
        for n in range(d2.N + 1):
            for f in SOFT_PFIELDS:
                out[f"{name}_p_s{n}_{f}"] = qp2.get_field(f, n)
            if n < d2.N:
                for f in ("A", "B", "b"):
                    out[f"{name}_p_s{n}_{f}"] = qp2.get_field(f, n)
        prep = mpcqp.solve_ocp_qp(qp2, ARG)
        for k, v in pack_report(prep).items():
            out[f"{name}_short_{k}"] = v
        pfull = mpcqp.partial_expand(prep.solution, pmap, qp)
        for k in ("y", "pi", "lam", "t"):
            out[f"{name}_pfull_{k}"] = getattr(pfull, k)
        print("soft", name, dq.nv, dq.ns, cmap.keep_x0, rep.iterations, d2.N, list(d2.ns),
              prep.iterations, flush=True)
    np.savez_compressed(HERE / "soft_cond.npz", **out)


# user-built dense QPs (qp_data.DenseQp, solve_dense_qp: solver.py:98-100)
DENSE_CASES = [(41, 6, 4, 2, 0), (42, 12, 8, 5, 3), (43, 20, 20, 10, 4), (44, 40, 30, 60, 0),
               (45, 9, 3, 0, 2)]
DENSE_MODES = (("speed8", "speed", 1e-8), ("balance6", "balance", 1e-6))


def dense_random_qp(lib, seed, nv, nb, ng, ns):
    """A feasible random dense QP (box, general and soft rows, one masked side)."""
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((nv, nv))
    q = lib.DenseQp(nv, 0, nb, ng, ns)
    q.set_field("H", F @ F.T + np.eye(nv))
    q.set_field("g", rng.standard_normal(nv))
    v0 = rng.uniform(-0.5, 0.5, nv)
    idxb = np.sort(rng.choice(nv, nb, replace=False)) if nb else np.zeros(0, dtype=int)
    if nb:
        q.set_field("idxb", idxb)
        q.set_field("lb", v0[idxb] - rng.uniform(0.1, 1.0, nb))
        q.set_field("ub", v0[idxb] + rng.uniform(0.1, 1.0, nb))
    if ng:
        C = rng.standard_normal((ng, nv))
        q.set_field("C", C)
        q.set_field("lg", C @ v0 - rng.uniform(0.1, 1.0, ng))
        q.set_field("ug", C @ v0 + rng.uniform(0.1, 1.0, ng))
    if ns:
        q.set_field("idxs", np.sort(rng.choice(nb + ng, ns, replace=False)))
        for f in ("Zl", "Zu"):
            q.set_field(f, rng.uniform(0.5, 2.0, ns))
        for f in ("zl", "zu"):
            q.set_field(f, rng.uniform(0.0, 1.0, ns))
    if nb + ng:
        mu = np.ones(nb + ng)
        mu[rng.integers(nb + ng)] = 0.0
        q.set_field("masku", mu)
    return q


def dense():
    out = {}
    for seed, nv, nb, ng, ns in DENSE_CASES:
        q = dense_random_qp(mpcqp, seed, nv, nb, ng, ns)
        for mname, preset, tol in DENSE_MODES:
            arg = mpcqp.mode_preset(preset).with_tol(tol)
            rep = mpcqp.solve_dense_qp(q, arg)
            for k, v in pack_report(rep).items():
                out[f"d{seed}_{mname}_{k}"] = v
            print("dense", seed, mname, rep.status.value, rep.iterations, flush=True)
    np.savez_compressed(HERE / "dense.npz", **out)


# dense QPs with equality constraints (kkt_dense.py:117-231): (seed, nv, ne, nb, ng,
# kkt_method, rank_deficient); speed mode, tol 1e-8
DENSE_EQ_CASES = [
    (61, 8, 2, 4, 2, "schur", False),
    (62, 12, 4, 6, 3, "schur", False),
    (63, 10, 3, 0, 4, "null_space", False),
    (64, 16, 5, 8, 0, "null_space", False),
    (65, 6, 6, 3, 1, "null_space", False),
    (66, 20, 8, 10, 5, "schur", False),
    (67, 20, 8, 10, 5, "null_space", False),
    (68, 9, 3, 4, 2, "schur", True),
    (69, 9, 3, 4, 2, "null_space", True),
]


def dense_eq_qp(lib, seed, nv, ne, nb, ng, rank_deficient=False):
    """A feasible random dense QP with ne equality rows A v = b (b = A v0)."""
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((nv, nv))
    q = lib.DenseQp(nv, ne, nb, ng, 0)
    q.set_field("H", F @ F.T + np.eye(nv))
    q.set_field("g", rng.standard_normal(nv))
    v0 = rng.uniform(-0.5, 0.5, nv)
    A = rng.standard_normal((ne, nv))
    if rank_deficient:
        A[-1] = 0.0   # an all-zero equality row: exactly singular for both methods
    q.set_field("A", A)
    q.set_field("b", A @ v0)
    if nb:
        idxb = np.sort(rng.choice(nv, nb, replace=False))
        q.set_field("idxb", idxb)
        q.set_field("lb", v0[idxb] - rng.uniform(0.1, 1.0, nb))
        q.set_field("ub", v0[idxb] + rng.uniform(0.1, 1.0, nb))
    if ng:
        C = rng.standard_normal((ng, nv))
        q.set_field("C", C)
        q.set_field("lg", C @ v0 - rng.uniform(0.1, 1.0, ng))
        q.set_field("ug", C @ v0 + rng.uniform(0.1, 1.0, ng))
    if nb + ng:
        mu = np.ones(nb + ng)
        mu[rng.integers(nb + ng)] = 0.0
        q.set_field("masku", mu)
    return q


def dense_eq():
    from dataclasses import replace

    out = {}
    for seed, nv, ne, nb, ng, method, rd in DENSE_EQ_CASES:
        q = dense_eq_qp(mpcqp, seed, nv, ne, nb, ng, rd)
        arg = replace(mpcqp.mode_preset("speed").with_tol(1e-8), kkt_method=method)
        rep = mpcqp.solve_dense_qp(q, arg)
        for k, v in pack_report(rep).items():
            out[f"e{seed}_{k}"] = v
        print("dense_eq", seed, method, rep.status.value, rep.iterations, rep.stats.flops, flush=True)
    np.savez_compressed(HERE / "dense_eq.npz", **out)


# modes beyond speed (ipm_core.py:131-168): (name, preset, tol, overrides)
MODES = [
    ("balance6", "balance", 1e-6, {}),
    ("balance8", "balance", 1e-8, {}),
    ("robust6", "robust", 1e-6, {}),
    ("sqrt8", "speed", 1e-8, {"riccati_variant": "square_root"}),
    ("abs8", "speed_abs", 1e-8, {}),
    ("sqrtbal6", "balance", 1e-6, {"riccati_variant": "square_root"}),
]
MODE_SOURCES = ([("r%d" % s, ("rnd", s)) for s, _ in RANDOM_CASES]
                + [("c0q0", ("cfg", 0, 0)), ("c1q1", ("cfg", 1, 1)), ("c1q2", ("cfg", 1, 2)),
                   ("c2q0", ("cfg", 2, 0)), ("c3q0", ("cfg", 3, 0)), ("c3q1", ("cfg", 3, 1))])
MODE_HEAVY = [("c4q56", ("cfg", 4, 56), ("balance6", "sqrt8", "robust6"))]


def mode_arg(name):
    import dataclasses

    for n, preset, tol, over in MODES:
        if n == name:
            return dataclasses.replace(mpcqp.mode_preset(preset).with_tol(tol), **over)
    raise KeyError(name)


def mode_source(src):
    if src[0] == "rnd":
        kw = dict(RANDOM_CASES)[src[1]]
        return qpgen.build_qp(mpcqp, *qpgen.random_ocp_fields(src[1], **kw))
    _, cfg, i = src
    return to_ref(make_batch(cfg, batch=1, start=i).qp(0))


def solve_modes():
    out = {}
    jobs = [(name, src, m) for name, src in MODE_SOURCES for m, *_ in MODES]
    jobs += [(name, src, m) for name, src, ms in MODE_HEAVY for m in ms]
    for name, src, m in jobs:
        rep = mpcqp.solve_ocp_qp(mode_source(src), mode_arg(m))
        for k, v in pack_report(rep).items():
            out[f"{name}_{m}_{k}"] = v
        print("modes", name, m, rep.status.value, rep.iterations, rep.stats.flops, flush=True)
    # ladders that end in Failure: the indefinite scalar LQR of known()
    for m, *_ in MODES:
        q = qpgen.scalar_lqr(mpcqp)
        q.set_field("r", 0, [1.0])
        q.set_field("R", 0, [[-1.0]])
        q.set_field("Q", 0, [[-1.0]])
        q.set_field("Q", 1, [[-1.0]])
        rep = mpcqp.solve_ocp_qp(q, mode_arg(m))
        out[f"indef_{m}_status"] = STATUS[rep.status.value]
        out[f"indef_{m}_iters"] = rep.iterations
        out[f"indef_{m}_flops"] = rep.stats.flops
    # RankDeficient escapes the QR factor in robust mode (linalg.py:180-184)
    for m, *_ in MODES:
        try:
            rep = mpcqp.solve_ocp_qp(qpgen.rank_deficient(mpcqp), mode_arg(m))
            out[f"rankdef_{m}_raised"] = 0
            for k, v in pack_report(rep).items():
                out[f"rankdef_{m}_{k}"] = v
        except mpcqp.errors.RankDeficient:
            out[f"rankdef_{m}_raised"] = 1
        print("rankdef", m, int(out[f"rankdef_{m}_raised"]), flush=True)
    np.savez_compressed(HERE / "modes.npz", **out)


# closed-loop MPC (mass_spring.py:222-273): (name, cfg kwargs, steps, preset, tol, warm)
CLOSED_LOOP_CASES = [
    ("m3", dict(masses=3, horizon=10), 8, "balance", 1e-6, "primal_dual"),
    ("m4", dict(masses=4, horizon=15, x0=[0.5, -0.3, 0.2, -0.6, 0.0, 0.0, 0.0, 0.0]), 6,
     "speed", 1e-8, "primal_dual"),
    ("m2", dict(masses=2, horizon=10), 5, "speed", 1e-8, "primal"),
]


def closed_loop():
    import mpcqp.mass_spring as ms

    out = {}
    for name, kw, steps, preset, tol, warm in CLOSED_LOOP_CASES:
        cfg = ms.MassSpringConfig(**kw)
        res = ms.run_closed_loop(cfg, steps, arg=mpcqp.mode_preset(preset).with_tol(tol),
                                 warm_start=warm, compare_cold=True)
        out[f"{name}_states"] = res.states
        out[f"{name}_inputs"] = res.inputs
        out[f"{name}_iters"] = np.array([r.iterations for r in res.records])
        out[f"{name}_cold_iters"] = np.array([r.cold_iterations for r in res.records])
        out[f"{name}_status"] = np.array([STATUS[r.status] for r in res.records])
        print("closed loop", name, out[f"{name}_iters"], out[f"{name}_cold_iters"], flush=True)
    # one shift on its own: solve m3's first QP, shift the solution
    cfg = ms.MassSpringConfig(masses=3, horizon=10)
    qp = ms.gen_mass_spring(cfg)
    rep = mpcqp.solve_ocp_qp(qp, mpcqp.mode_preset("balance").with_tol(1e-6))
    g = ms._shift_guess(qp, make_view(qp), rep.solution, cfg.horizon)
    for k in ("y", "pi", "lam", "t"):
        out[f"shift_sol_{k}"] = getattr(rep.solution, k)
        out[f"shift_guess_{k}"] = getattr(g, k)
    np.savez_compressed(HERE / "closed_loop.npz", **out)


def qp_files():
    """Reference-written QP text files and CLI reports (qp_io.py, cli.py)."""
    import subprocess

    d = HERE / "qp_files"
    d.mkdir(exist_ok=True)
    s, kw = RANDOM_CASES[1]
    mpcqp.qp_write(str(d / "rand12.qp"), qpgen.build_qp(mpcqp, *qpgen.random_ocp_fields(s, **kw)))
    env = {"PYTHONPATH": "/root/reference/pkg/src", "PATH": "/usr/bin:/bin"}
    py = sys.executable
    subprocess.run([py, "-m", "mpcqp.cli", "gen-mass-spring", "--masses", "3", "--horizon", "6",
                    "--out", str(d / "mass3.qp")], check=True, env=env, cwd=str(d))
    for name, extra in (("mass3_balance", []), ("mass3_speed", ["--mode", "speed", "--tol", "1e-8"]),
                        ("mass3_partial", ["--path", "partial:2"]),
                        ("mass3_condense", ["--path", "condense"])):
        r = subprocess.run([py, "-m", "mpcqp.cli", "solve", "--qp", "mass3.qp", *extra],
                           env=env, cwd=str(d), capture_output=True, text=True)
        (d / f"{name}.report").write_text(r.stdout)
        print(name, r.returncode, flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["known", "residuals", "newton", "solve_random", "solve_cfg", "pcond",
                            "solve_modes", "closed_loop", "qp_files", "fcond", "soft_cond", "dense",
                            "pcond_full", "dense_eq", "fcond_sqrt"]
    for w in which:
        globals()[w]()
