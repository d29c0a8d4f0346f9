"""Closed-loop MPC on the spring-chain benchmark with shifted warm starts.

Drop-in for the reference's mass_spring module drivers (MassSpringConfig,
gen_mass_spring, mass_spring_dynamics, default_x0, run_closed_loop;
mass_spring.py:55-273), B200-first: the controller solve is the fused GPU IPM
(any mode; the reference's default is ``balance`` at tol 1e-6) and the
solution shift that seeds the next solve (``_shift_guess``,
mass_spring.py:152-195) is a CUDA kernel behind the C ABI
(``ocpqp_shift_guess``).  :func:`run_closed_loop_batch` runs many plants in
lockstep -- one batched solve, one shift launch and one plant update per
step, every array device resident.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from .batch import OcpQpBatch
from .errors import ClosedLoopFailed, InvalidConfig
from .generators import chain_dynamics
from .ipm import Status, mode_preset
from .qp_data import OcpQp, OcpQpDim
from .solver import _torch, get_plan, solve_ocp_qp_batch

__all__ = ["MassSpringConfig", "default_x0", "mass_spring_dynamics", "gen_mass_spring",
           "StepRecord", "ClosedLoopResult", "shift_guess", "run_closed_loop",
           "run_closed_loop_batch"]


@dataclass
class MassSpringConfig:
    """Benchmark configuration (mass_spring.py:55-85): M unit masses, the first
    M - 1 actuated, sampling time ``ts``, |u| <= u_bound, |x| <= x_bound."""

    masses: int = 2
    horizon: int = 10
    ts: float = 0.5
    x0: object = None
    u_bound: float = 0.5
    x_bound: float = 4.0

    def validate(self):
        if self.masses < 2:
            raise InvalidConfig("need at least 2 masses")
        if self.horizon < 1:
            raise InvalidConfig("horizon must be >= 1")
        if self.ts <= 0.0:
            raise InvalidConfig("sampling time must be > 0")
        if self.u_bound <= 0.0 or self.x_bound <= 0.0:
            raise InvalidConfig("bounds must be > 0")
        if self.x0 is not None:
            x0 = np.asarray(self.x0, dtype=float)
            if x0.shape != (2 * self.masses,):
                raise InvalidConfig(f"x0 must have {2 * self.masses} entries, got {x0.shape}")
            if np.any(np.abs(x0) > self.x_bound):
                raise InvalidConfig("x0 violates the state bounds")
        return self


def default_x0(masses):
    """Alternating-position rest state of amplitude 0.6 (mass_spring.py:88-96)."""
    x0 = np.zeros(2 * masses)
    x0[:masses] = 0.6 * (-1.0) ** np.arange(masses)
    return x0


def mass_spring_dynamics(masses, ts):
    """Exactly discretised (A, B), first M - 1 masses actuated (mass_spring.py:99-114)."""
    return chain_dynamics(masses, ts, tuple(range(masses - 1)))


def gen_mass_spring(cfg):
    """The benchmark OCP QP of one configuration (mass_spring.py:117-149)."""
    cfg.validate()
    M, N = cfg.masses, cfg.horizon
    nx, nu = 2 * M, M - 1
    A, B = mass_spring_dynamics(M, cfg.ts)
    x0 = np.asarray(cfg.x0, dtype=float) if cfg.x0 is not None else default_x0(M)
    dim = OcpQpDim(N, nx=[nx] * (N + 1), nu=[nu] * N + [0], nb=[nu + nx] * N + [nx],
                   ng=[0] * (N + 1), ns=[0] * (N + 1))
    qp = OcpQp(dim)
    lb = np.concatenate([-cfg.u_bound * np.ones(nu), -cfg.x_bound * np.ones(nx)])
    for n in range(N):
        qp.set_field("A", n, A)
        qp.set_field("B", n, B)
        qp.set_field("Q", n, np.eye(nx))
        qp.set_field("R", n, np.eye(nu))
        qp.set_field("idxb", n, np.arange(nu + nx))
        qp.set_field("lb", n, lb)
        qp.set_field("ub", n, -lb)
    qp.set_field("Q", N, np.eye(nx))
    qp.set_field("idxb", N, np.arange(nx))
    qp.set_field("lb", N, -cfg.x_bound * np.ones(nx))
    qp.set_field("ub", N, cfg.x_bound * np.ones(nx))
    qp.set_field("lbx", 0, x0)
    qp.set_field("ubx", 0, x0)
    return qp


@dataclass
class StepRecord:
    step: int
    status: str
    iterations: int
    cold_iterations: object = None


@dataclass
class ClosedLoopResult:
    records: list
    states: np.ndarray     # (steps + 1, nx)
    inputs: np.ndarray     # (steps, nu)

    @property
    def total_iterations(self):
        return sum(r.iterations for r in self.records)

    @property
    def total_cold_iterations(self):
        vals = [r.cold_iterations for r in self.records]
        return None if any(v is None for v in vals) else sum(vals)


def shift_guess(batch, sol, out=None, stream=None):
    """Batched ``_shift_guess`` (mass_spring.py:152-195) on the device.

    ``batch`` is a device-resident OcpQpBatch, ``sol`` the (y, pi, lam, t)
    device tensors of its solutions; returns the shifted guesses (new tensors
    unless ``out`` is given).
    """
    torch = _torch()
    y, pi, lam, t = sol
    if out is None:
        out = tuple(torch.empty_like(a) for a in (y, pi, lam, t))
    plan = get_plan(batch)
    dc = nat.data_c(batch)
    si = nat.OcpIterC(y.data_ptr(), pi.data_ptr(), lam.data_ptr(), t.data_ptr())
    go = nat.OcpIterC(*(a.data_ptr() for a in out))
    s = stream if stream is not None else torch.cuda.current_stream()
    nat.check(nat.lib().ocpqp_shift_guess(plan.handle, ctypes.byref(dc), ctypes.byref(si),
                                          ctypes.byref(go), ctypes.c_void_p(s.cuda_stream)))
    return out


def _x0_rows(batch):
    """Box rows of stage 0 that fix the initial state: (row index, state component)."""
    d = batch.dim
    nu0 = int(d.nu[0])
    idxb0 = np.asarray(batch.idxb[0])
    rows = [(i, int(k) - nu0) for i, k in enumerate(idxb0) if int(k) >= nu0]
    return np.array([r for r, _ in rows], dtype=np.int64), np.array([c for _, c in rows],
                                                                    dtype=np.int64)


def run_closed_loop_batch(cfg, x0s, steps, arg=None, warm_start="primal_dual",
                          compare_cold=False, strict=True, device="cuda", graph=True):
    """Closed-loop MPC of B independent chains (same model, own initial states).

    Per step: impose every plant's state through the stage-0 box rows, solve
    the whole batch (warm started from the shifted previous solutions after
    the first step), apply each first input to its exact discrete plant, shift
    the solutions on the device.  Every buffer is preallocated, so with
    ``graph`` the warm steps are one captured CUDA graph replayed per step
    (the step is launch-bound: the index writes, the solve's kernels, the
    shift and the plant update); the first (cold) step and the capture's
    warm-up step run eagerly.  Returns a list of ClosedLoopResult, one per
    plant.  With ``strict`` a non-Success controller solve raises
    ClosedLoopFailed for the first failing step (the reference's behaviour,
    mass_spring.py:256-260); otherwise the records carry the statuses.
    """
    torch = _torch()
    cfg.validate()
    if steps < 1:
        raise InvalidConfig("steps must be >= 1")
    arg = arg or mode_preset("balance").with_tol(1e-6)
    x0s = np.atleast_2d(np.asarray(x0s, dtype=float))
    Bn = x0s.shape[0]
    M = cfg.masses
    nx, nu = 2 * M, M - 1
    A, Bm = mass_spring_dynamics(M, cfg.ts)
    host = OcpQpBatch.from_qps([gen_mass_spring(replace(cfg, x0=x0s[0]))])
    batch = OcpQpBatch(host.dim, Bn, idxb=host.idxb, idxs=host.idxs)
    for name, arr in host.fields.items():
        per_qp = name in ("lb", "ub")
        batch.alloc(name, per_qp, 0.0)
        batch.fields[name][:] = arr
    dev = batch.to(device)
    lay = batch.layout
    rows, comps = _x0_rows(batch)
    off = int(lay.stage_slice("lb", 0).start)
    cols = torch.as_tensor(off + rows, device=device)
    comps_t = torch.as_tensor(comps, device=device)
    f64 = dict(dtype=torch.float64, device=device)
    At = torch.as_tensor(A.T.copy(), **f64)
    Bt = torch.as_tensor(Bm.T.copy(), **f64)
    x = torch.as_tensor(x0s, **f64).clone()
    u_off0 = int(lay.u_off[0])

    def buffers():
        return dict(y=torch.empty((Bn, lay.ny), **f64), pi=torch.empty((Bn, lay.ne), **f64),
                    lam=torch.empty((Bn, lay.nc), **f64), t=torch.empty((Bn, lay.nc), **f64),
                    status=torch.empty(Bn, dtype=torch.int32, device=device),
                    iters=torch.empty(Bn, dtype=torch.int32, device=device),
                    res=torch.empty((Bn, 5), **f64),
                    flops=torch.empty(Bn, dtype=torch.int64, device=device), trace=None)

    out = buffers()
    cold = buffers() if compare_cold else None
    guess = tuple(torch.zeros_like(out[k]) for k in ("y", "pi", "lam", "t"))
    hist_x = torch.empty((steps + 1, Bn, nx), **f64)
    hist_u = torch.empty((steps, Bn, nu), **f64)
    hist_st = torch.empty((steps, Bn), dtype=torch.int32, device=device)
    hist_it = torch.empty((steps, Bn), dtype=torch.int32, device=device)
    hist_cold = torch.empty((steps, Bn), dtype=torch.int32, device=device) if compare_cold else None
    hist_x[0].copy_(x)
    cold_arg = replace(arg, warm_start="none")
    warm_arg = replace(arg, warm_start=warm_start)

    def step(first):
        s = torch.cuda.current_stream()
        xs = x[:, comps_t]
        dev.fields["lb"][:, cols] = xs
        dev.fields["ub"][:, cols] = xs
        solve_ocp_qp_batch(dev, cold_arg if first else warm_arg, guess=None if first else guess,
                           trace=False, out=out, stream=s)
        if compare_cold:
            solve_ocp_qp_batch(dev, cold_arg, trace=False, out=cold, stream=s)
        u0 = out["y"][:, u_off0:u_off0 + nu]
        x.copy_(x @ At + u0 @ Bt)
        shift_guess(dev, (out["y"], out["pi"], out["lam"], out["t"]), out=guess, stream=s)

    def record(k):
        hist_u[k].copy_(out["y"][:, u_off0:u_off0 + nu])
        hist_x[k + 1].copy_(x)
        hist_st[k].copy_(out["status"])
        hist_it[k].copy_(out["iters"])
        if compare_cold:
            hist_cold[k].copy_(cold["iters"])

    step(True)
    record(0)
    k = 1
    if graph and steps > 2:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):   # warm-up of the warm step (a real step)
                step(False)
                record(1)
            torch.cuda.current_stream().wait_stream(side)
            k = 2
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(False)
            while k < steps:
                g.replay()
                record(k)
                k += 1
        except RuntimeError as exc:   # capture unsupported here: the rest runs eagerly
            import warnings

            warnings.warn(f"closed loop: CUDA graph capture failed ({exc}); running eagerly")
            torch.cuda.synchronize()
    while k < steps:
        step(False)
        record(k)
        k += 1
    torch.cuda.synchronize()
    st = hist_st.cpu().numpy()
    its = hist_it.cpu().numpy()
    if strict:
        bad = np.argwhere(st != 0)
        if bad.size:
            kk, i = (int(v) for v in bad[np.argmin(bad[:, 0])])
            code = int(st[kk, i])
            names = ["Success", "MaxIter", "MinStep", "NaNDetected", "Failure"]
            raise ClosedLoopFailed(
                f"controller solve failed at step {kk} (plant {i}) with status "
                f"{names[code] if 0 <= code < 5 else code}", step=kk)
    S = hist_x.permute(1, 0, 2).cpu().numpy()
    U = hist_u.permute(1, 0, 2).cpu().numpy()
    cs = hist_cold.cpu().numpy() if compare_cold else None
    names = {int(c): s.value for c, s in zip(range(5), (Status.Success, Status.MaxIter,
                                                         Status.MinStep, Status.NaNDetected,
                                                         Status.Failure))}
    results = []
    for i in range(Bn):
        recs = [StepRecord(step=k2, status=names.get(int(st[k2, i]), str(int(st[k2, i]))),
                           iterations=int(its[k2, i]),
                           cold_iterations=int(cs[k2, i]) if compare_cold else None)
                for k2 in range(steps)]
        results.append(ClosedLoopResult(records=recs, states=S[i], inputs=U[i]))
    return results


def run_closed_loop(cfg, steps, arg=None, warm_start="primal_dual", compare_cold=False):
    """Drop-in for mass_spring.run_closed_loop (mass_spring.py:222-273): one
    plant, the GPU solve and the device shift at every step."""
    cfg.validate()
    x = np.asarray(cfg.x0, dtype=float) if cfg.x0 is not None else default_x0(cfg.masses)
    return run_closed_loop_batch(cfg, x[None], steps, arg=arg, warm_start=warm_start,
                                 compare_cold=compare_cold, strict=True)[0]
