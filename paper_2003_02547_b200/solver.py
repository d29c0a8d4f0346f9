"""Drop-in solve entry points over the CUDA library.

* :func:`solve_ocp_qp` -- the reference's single-QP call
  ``solve_ocp_qp(qp, arg=None, guess=None) -> SolveReport``
  (mpcqp/solver.py:103-105), same objects in and out;
* :func:`solve_ocp_qp_batch` -- the batched form over a packed
  :class:`OcpQpBatch` (or a list of ``OcpQp``), device-resident, one fused
  kernel launch for the whole batch;
* :func:`solve_ocp_qp_host` -- the same over host buffers through the C ABI's
  ``ocpqp_solve_host`` (copies in, solve, copies out): the end-to-end path an
  FFI binding of the reference takes;
* :func:`newton_step` / :func:`compute_residuals` -- the backend plug-in
  points (riccati_factor + solve, kkt_ocp.py:142-320; view.residuals,
  view.py:272-288) exposed batched for parity testing.

Every path runs on the GPU; a missing library raises NativeLibraryError.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .batch import OcpQpBatch
from .errors import DimensionMismatch, NonPositiveIterate, RankDeficient, SingularSlackBlock
from .ipm import STATUS_CODES, IpmArg, IterRecord, SolverStats, Status, supported_reason
from .layout import QpResiduals, QpSolution
from .qp_data import OcpQp, errors_only, validate

__all__ = ["SolveReport", "BatchReport", "solve_ocp_qp", "solve_ocp_qp_batch",
           "solve_ocp_qp_host", "newton_step", "compute_residuals", "get_plan"]

_PLANS = {}
_MAX_PLANS = 8   # least-recently-used plans beyond this are released


def _device_index(batch, device=None):
    for arr in batch.fields.values():
        dev = getattr(arr, "device", None)
        if dev is not None and getattr(dev, "type", "") == "cuda":
            return dev.index if dev.index is not None else 0
    if device is not None:
        import torch

        d = torch.device(device)
        if d.type == "cuda":
            return d.index if d.index is not None else torch.cuda.current_device()
    import torch

    return torch.cuda.current_device()


def get_plan(batch: OcpQpBatch, device=None):
    """Cached plan for the batch's structure, size and CUDA device.

    A plan owns one workspace: solves on it are stream-ordered (one solve in
    flight per plan, the C ABI's contract).  The plan is created on, and its
    solves run on, the device that holds the batch."""
    import torch

    dev = _device_index(batch, device)
    key = (batch.structure_key(), batch.B, dev)
    plan = _PLANS.pop(key, None)
    if plan is None:
        with torch.cuda.device(dev):
            plan = nat.Plan(batch, batch.B)
        while len(_PLANS) >= _MAX_PLANS:
            old = _PLANS.pop(next(iter(_PLANS)))
            old.close()
    _PLANS[key] = plan   # most recently used last
    return plan


@dataclass
class SolveReport:
    """Solution, statistics and final residuals (solver.py:63-77)."""

    solution: QpSolution
    stats: SolverStats
    residuals: object

    @property
    def status(self):
        return self.stats.status

    @property
    def iterations(self):
        return self.stats.iterations


def _check_arg(arg):
    arg = (arg or IpmArg()).validate()
    why = supported_reason(arg)
    if why is not None:
        raise NotImplementedError(f"unsupported IpmArg setting: {why}")
    return arg


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .errors import NativeLibraryError

        raise NativeLibraryError("no CUDA device: the solver has no CPU fallback")
    return torch


def _as_batch(qps_or_batch, check=True):
    if isinstance(qps_or_batch, OcpQpBatch):
        return qps_or_batch
    if isinstance(qps_or_batch, OcpQp):
        qps_or_batch = [qps_or_batch]
    qps = list(qps_or_batch)
    if check:
        for q in qps:
            bad = errors_only(validate(q))
            if bad:
                raise ValueError("QP fails validation: " + "; ".join(str(v) for v in bad))
    return OcpQpBatch.from_qps(qps)


def _on_device(batch, device):
    torch = _torch()
    for arr in batch.fields.values():
        if not (isinstance(arr, torch.Tensor) and arr.is_cuda):
            return batch.to(device)
    return batch


class BatchReport:
    """Struct-of-arrays outcome of a batched solve (tensors stay on the device)."""

    def __init__(self, batch, arg, y, pi, lam, t, status, iters, res, flops, trace):
        self.batch = batch
        self.arg = arg
        self.y, self.pi, self.lam, self.t = y, pi, lam, t
        self.status_code = status
        self.iterations = iters
        self.res = res
        self.flops = flops
        self.trace = trace
        self._host = None

    def _h(self):
        if self._host is None:
            def h(x):
                if x is None:
                    return None
                return x if isinstance(x, np.ndarray) else x.detach().cpu().numpy()
            self._host = {k: h(getattr(self, k)) for k in
                          ("y", "pi", "lam", "t", "status_code", "iterations", "res", "flops",
                           "trace")}
        return self._host

    def statuses(self):
        return [STATUS_CODES.get(int(c), c) for c in self._h()["status_code"]]

    def report(self, i, residual_vectors=True) -> SolveReport:
        """The reference-style SolveReport of QP ``i``."""
        h = self._h()
        code = int(h["status_code"][i])
        if code == 5:
            raise NonPositiveIterate("lam, t must be > 0 on active rows")
        if code == 6:
            raise SingularSlackBlock("augmented soft-slack diagonal must be > 0")
        if code == 7:
            raise RankDeficient("QR array algorithm: rank-deficient stage stack")
        lay = self.batch.layout
        sol = QpSolution(lay, h["y"][i].copy(), h["pi"][i].copy(), h["lam"][i].copy(),
                         h["t"][i].copy())
        it = int(h["iterations"][i])
        trace = []
        if h["trace"] is not None:
            for k in range(min(it, h["trace"].shape[1])):
                r = h["trace"][i, k]
                trace.append(IterRecord(k, float(r[0]), float(r[1]), float(r[2]), float(r[3]),
                                        float(r[4]), float(r[5]), float(r[6]), float(r[7])))
        res = h["res"][i]
        stats = SolverStats(status=STATUS_CODES[code], iterations=it, res_g=float(res[0]),
                            res_b=float(res[1]), res_d=float(res[2]), res_m=float(res[3]),
                            mu=float(res[4]), flops=int(h["flops"][i]), trace=trace)
        residuals = None
        if residual_vectors:
            residuals = compute_residuals(self.batch.select([i]) if self.batch.B > 1 else self.batch,
                                          sol)
        return SolveReport(solution=sol, stats=stats, residuals=residuals)


def _guess_arrays(guess, batch, torch, device):
    lay = batch.layout
    B = batch.B
    if isinstance(guess, BatchReport):
        parts = (guess.y, guess.pi, guess.lam, guess.t)
    elif isinstance(guess, QpSolution):
        parts = tuple(np.asarray(a)[None] for a in (guess.y, guess.pi, guess.lam, guess.t))
    elif isinstance(guess, (list, tuple)) and guess and isinstance(guess[0], QpSolution):
        parts = tuple(np.stack([np.asarray(getattr(g, k)) for g in guess])
                      for k in ("y", "pi", "lam", "t"))
    else:
        parts = tuple(guess)
    out = []
    for a, n in zip(parts, (lay.ny, lay.ne, lay.nc, lay.nc)):
        ta = torch.as_tensor(a, dtype=torch.float64, device=device).reshape(-1, n)
        if ta.shape[0] != B:
            raise DimensionMismatch("guess does not match QP dimensions")
        out.append(ta.clone())
    return out


def solve_ocp_qp_batch(batch, arg=None, guess=None, device="cuda", trace=True,
                       stream=None, out=None, phase_debug=None) -> BatchReport:
    """Solve every QP of a batch with the fused GPU IPM (one kernel launch).

    ``phase_debug`` (diagnostics): an int64 device tensor [B, 8] receiving the
    clock64 cycles each QP spent in residuals / factor / affine solve /
    corrector solve(s) / step+update, the total and the iteration count.
    """
    arg = _check_arg(arg)
    torch = _torch()
    batch = _as_batch(batch)
    dev_batch = _on_device(batch, device)
    lay = batch.layout
    B = batch.B
    plan = get_plan(dev_batch)
    f64 = dict(dtype=torch.float64, device=device)
    if out is None:
        out = dict(
            y=torch.empty((B, lay.ny), **f64), pi=torch.empty((B, lay.ne), **f64),
            lam=torch.empty((B, lay.nc), **f64), t=torch.empty((B, lay.nc), **f64),
            status=torch.empty(B, dtype=torch.int32, device=device),
            iters=torch.empty(B, dtype=torch.int32, device=device),
            res=torch.empty((B, 5), **f64),
            flops=torch.empty(B, dtype=torch.int64, device=device),
            trace=torch.zeros((B, max(1, arg.iter_max), 8), **f64) if trace else None,
        )
    s = stream if stream is not None else torch.cuda.current_stream(device)
    if arg.warm_start != "none" and guess is not None:
        # the guess lands in the output buffers on the solve's stream
        with torch.cuda.stream(s):
            gy, gpi, glam, _ = _guess_arrays(guess, batch, torch, device)
            out["y"].copy_(gy)
            if arg.warm_start == "primal_dual":
                out["pi"].copy_(gpi)
                out["lam"].copy_(glam)
        carg = nat.arg_to_c(arg)
    else:
        from dataclasses import replace
        carg = nat.arg_to_c(replace(arg, warm_start="none"))
    dc = nat.data_c(dev_batch)
    it = nat.OcpIterC(out["y"].data_ptr(), out["pi"].data_ptr(), out["lam"].data_ptr(),
                      out["t"].data_ptr())
    st = nat.OcpStatsC(out["status"].data_ptr(), out["iters"].data_ptr(), out["res"].data_ptr(),
                       out["flops"].data_ptr(),
                       out["trace"].data_ptr() if out["trace"] is not None else None)
    if phase_debug is not None or getattr(plan, "_dbg_on", False):
        L = nat.lib()
        L.ocpqp_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        nat.check(L.ocpqp_debug_phases(plan.handle, None if phase_debug is None
                                       else ctypes.c_void_p(phase_debug.data_ptr())))
        plan._dbg_on = phase_debug is not None
    nat.check(nat.lib().ocpqp_solve(plan.handle, ctypes.byref(dc), ctypes.byref(carg),
                                    ctypes.byref(it), ctypes.byref(st),
                                    ctypes.c_void_p(s.cuda_stream)))
    return BatchReport(dev_batch, arg, out["y"], out["pi"], out["lam"], out["t"], out["status"],
                       out["iters"], out["res"], out["flops"], out["trace"])


def solve_ocp_qp_host(batch, arg=None, trace=False, out=None, stream=None) -> BatchReport:
    """Host-buffer solve through ``ocpqp_solve_host`` (H2D, solve, D2H inside)."""
    arg = _check_arg(arg)
    torch = _torch()
    batch = _as_batch(batch)
    lay = batch.layout
    B = batch.B
    plan = get_plan(batch)
    if out is None:
        out = dict(
            y=np.empty((B, lay.ny)), pi=np.empty((B, lay.ne)), lam=np.empty((B, lay.nc)),
            t=np.empty((B, lay.nc)), status=np.empty(B, dtype=np.int32),
            iters=np.empty(B, dtype=np.int32), res=np.empty((B, 5)),
            flops=np.empty(B, dtype=np.int64),
            trace=np.zeros((B, max(1, arg.iter_max), 8)) if trace else None)
    from dataclasses import replace
    carg = nat.arg_to_c(replace(arg, warm_start="none"))
    dc = nat.data_c(batch)
    P = nat.ptr_of
    it = nat.OcpIterC(P(out["y"]), P(out["pi"]), P(out["lam"]), P(out["t"]))
    st = nat.OcpStatsC(P(out["status"]), P(out["iters"]), P(out["res"]), P(out["flops"]),
                       P(out["trace"]))
    s = stream if stream is not None else torch.cuda.current_stream()
    nat.check(nat.lib().ocpqp_solve_host(plan.handle, ctypes.byref(dc), ctypes.byref(carg),
                                         ctypes.byref(it), ctypes.byref(st),
                                         ctypes.c_void_p(s.cuda_stream)))
    return BatchReport(batch, arg, out["y"], out["pi"], out["lam"], out["t"], out["status"],
                       out["iters"], out["res"], out["flops"], out["trace"])


def solve_ocp_qp(qp, arg=None, guess=None) -> SolveReport:
    """Solve one optimal-control QP (drop-in for mpcqp.solve_ocp_qp)."""
    arg = _check_arg(arg)
    batch = _as_batch([qp])
    if guess is not None:
        if guess.y.shape[0] != batch.layout.ny or guess.lam.shape[0] != batch.layout.nc:
            raise DimensionMismatch("guess does not match QP dimensions")
    rep = solve_ocp_qp_batch(batch, arg, guess=guess if guess is not None else None)
    return rep.report(0)


def compute_residuals(qp_or_batch, solution, device="cuda"):
    """KKT residuals of a point (view.compute_residuals, view.py:698-706).

    ``solution`` is a QpSolution (single QP) or a tuple of [B, n] arrays.
    Returns a QpResiduals (single) or a dict of device tensors (batched).
    """
    torch = _torch()
    single = isinstance(solution, QpSolution)
    batch = _as_batch(qp_or_batch, check=False)
    dev = _on_device(batch, device)
    lay = batch.layout
    B = batch.B
    if single:
        parts = (solution.y, solution.pi, solution.lam, solution.t)
    else:
        parts = solution
    f64 = dict(dtype=torch.float64, device=device)
    y, pi, lam, t = (torch.as_tensor(np.asarray(a) if isinstance(a, np.ndarray) else a, **f64)
                     .reshape(B, -1).contiguous() for a in parts)
    rg = torch.empty((B, lay.ny), **f64)
    rb = torch.empty((B, lay.ne), **f64)
    rd = torch.empty((B, lay.nc), **f64)
    rm = torch.empty((B, lay.nc), **f64)
    norms = torch.empty((B, 5), **f64)
    plan = get_plan(dev)
    dc = nat.data_c(dev)
    pt = nat.OcpIterC(y.data_ptr(), pi.data_ptr(), lam.data_ptr(), t.data_ptr())
    s = torch.cuda.current_stream(device)
    nat.check(nat.lib().ocpqp_residuals(plan.handle, ctypes.byref(dc), ctypes.byref(pt),
                                        rg.data_ptr(), rb.data_ptr(), rd.data_ptr(), rm.data_ptr(),
                                        norms.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
    if not single:
        return dict(r_g=rg, r_b=rb, r_d=rd, r_m=rm, norms=norms)
    n = norms[0].cpu().numpy()
    return QpResiduals(r_g=rg[0].cpu().numpy(), r_b=rb[0].cpu().numpy(), r_d=rd[0].cpu().numpy(),
                       r_m=rm[0].cpu().numpy(), res_g=float(n[0]), res_b=float(n[1]),
                       res_d=float(n[2]), res_m=float(n[3]), mu=float(n[4]))


def newton_step(batch, iterate, r_g, r_b, r_d, r_m, reg=0.0, device="cuda"):
    """Batched classical Riccati factor + solve at an iterate.

    ``iterate`` is (y, pi, lam, t) of [B, n] arrays (only lam, t are read).
    Returns ((dy, dpi, dlam, dt), fail_stage) with fail_stage[i] = -1 on
    success, the FactorizationFailed stage otherwise (-2 / -3 for the
    NonPositiveIterate / SingularSlackBlock raises of the reference).
    """
    torch = _torch()
    batch = _as_batch(batch, check=False)
    dev = _on_device(batch, device)
    lay = batch.layout
    B = batch.B
    f64 = dict(dtype=torch.float64, device=device)

    def T(a, n):
        return torch.as_tensor(np.asarray(a) if isinstance(a, np.ndarray) else a,
                               **f64).reshape(B, n).contiguous()

    _, _, lam, t = iterate
    lam, t = T(lam, lay.nc), T(t, lay.nc)
    rg, rb, rd, rm = T(r_g, lay.ny), T(r_b, lay.ne), T(r_d, lay.nc), T(r_m, lay.nc)
    dy = torch.empty((B, lay.ny), **f64)
    dpi = torch.empty((B, lay.ne), **f64)
    dl = torch.empty((B, lay.nc), **f64)
    dt = torch.empty((B, lay.nc), **f64)
    fail = torch.empty(B, dtype=torch.int32, device=device)
    plan = get_plan(dev)
    dc = nat.data_c(dev)
    it = nat.OcpIterC(None, None, lam.data_ptr(), t.data_ptr())
    stp = nat.OcpIterC(dy.data_ptr(), dpi.data_ptr(), dl.data_ptr(), dt.data_ptr())
    s = torch.cuda.current_stream(device)
    nat.check(nat.lib().ocpqp_newton_step(plan.handle, ctypes.byref(dc), float(reg),
                                          ctypes.byref(it), rg.data_ptr(), rb.data_ptr(),
                                          rd.data_ptr(), rm.data_ptr(), ctypes.byref(stp),
                                          fail.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
    return (dy, dpi, dl, dt), fail
