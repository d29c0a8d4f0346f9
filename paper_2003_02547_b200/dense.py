"""Dense QP type and its solve (reference qp_data.DenseQp, qp_data.py:426-500;
solver.solve_dense_qp, solver.py:98-100).

Dense QPs with equality constraints (ne > 0) run on their own kernel
(csrc/ocpqp_dense.cu, C ABI ocpqp_dense_*) with the reference's two equality
methods, IpmArg.kkt_method "schur" (Schur complement A Hred^-1 A' + reg_dual I)
and "null_space" (Householder QR of A', reduced Hessian on the null-space
basis), kkt_dense.py:117-231 -- speed-mode loop, no soft rows (other modes
raise NotImplementedError).

A dense QP without equality constraints (ne = 0, the form full condensing
produces, condensing.py:297) is the single-stage optimal-control QP with
N = 0, nx = 0, nu = nv: H -> R, g -> r, C -> D, the box / general / soft rows
unchanged.  On that form the reference's dense backend (kkt_dense.py:117-256:
Hred = H + C' diag(gamma) C, Cholesky, dv = -Hred^-1 rhat) and its Riccati
backend at N = 0 perform the same operations in the same order -- same
iterates, same iteration counts and the same counted flops (checked against
the reference in tests/golden/fcond.npz) -- so the dense QP is solved by the
same fused sm_100a kernels as every OCP-QP.
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch, IndexOutOfRange, InvalidDim, UnknownField
from .qp_data import OcpQp, OcpQpDim

__all__ = ["DenseQp", "dense_to_ocp", "ocp_to_dense", "solve_dense_qp", "solve_dense_qp_batch",
           "DenseLayout"]

_SHAPES = {
    "H": lambda q: (q.nv, q.nv), "g": lambda q: (q.nv,),
    "A": lambda q: (q.ne, q.nv), "b": lambda q: (q.ne,),
    "idxb": lambda q: (q.nb,), "lb": lambda q: (q.nb,), "ub": lambda q: (q.nb,),
    "C": lambda q: (q.ng, q.nv), "lg": lambda q: (q.ng,), "ug": lambda q: (q.ng,),
    "idxs": lambda q: (q.ns,), "Zl": lambda q: (q.ns,), "Zu": lambda q: (q.ns,),
    "zl": lambda q: (q.ns,), "zu": lambda q: (q.ns,), "sl_lb": lambda q: (q.ns,),
    "su_lb": lambda q: (q.ns,),
    "maskl": lambda q: (q.nb + q.ng,), "masku": lambda q: (q.nb + q.ng,),
}
_INT = ("idxb", "idxs")
# dense field -> stage-0 field of the N = 0 OCP form
_TO_OCP = {"H": "R", "g": "r", "idxb": "idxb", "lb": "lb", "ub": "ub", "C": "D", "lg": "lg",
           "ug": "ug", "idxs": "idxs", "Zl": "Zl", "Zu": "Zu", "zl": "zl", "zu": "zu",
           "sl_lb": "sl_lb", "su_lb": "su_lb", "maskl": "maskl", "masku": "masku"}


class DenseQp:
    """Dense QP over nv variables, zero-initialised (qp_data.py:426-500).

    Fields: H g A b idxb lb ub C lg ug idxs Zl Zu zl zu sl_lb su_lb maskl
    masku; ``idxb`` selects the box-constrained components of v; the masks
    cover the nb + ng constraint rows (box rows first).
    """

    kind = "dense"

    def __init__(self, nv, ne=0, nb=0, ng=0, ns=0):
        for name, val in (("nv", nv), ("ne", ne), ("nb", nb), ("ng", ng), ("ns", ns)):
            if int(val) < 0:
                raise InvalidDim(f"{name} must be >= 0")
        if nb > nv:
            raise InvalidDim(f"nb = {nb} exceeds nv = {nv}")
        if ns > nb + ng:
            raise InvalidDim(f"ns = {ns} exceeds nb + ng = {nb + ng}")
        self.nv, self.ne, self.nb, self.ng, self.ns = int(nv), int(ne), int(nb), int(ng), int(ns)
        inf = np.inf
        self._data = {
            "H": np.zeros((nv, nv)), "g": np.zeros(nv), "A": np.zeros((ne, nv)), "b": np.zeros(ne),
            "idxb": np.arange(nb, dtype=int), "lb": np.full(nb, -inf), "ub": np.full(nb, inf),
            "C": np.zeros((ng, nv)), "lg": np.full(ng, -inf), "ug": np.full(ng, inf),
            "idxs": np.arange(ns, dtype=int), "Zl": np.zeros(ns), "Zu": np.zeros(ns),
            "zl": np.zeros(ns), "zu": np.zeros(ns), "sl_lb": np.zeros(ns), "su_lb": np.zeros(ns),
            "maskl": np.ones(nb + ng), "masku": np.ones(nb + ng),
        }
        self._rev = 0

    def field_names(self):
        return sorted(_SHAPES)

    def set_field(self, name, value, stage=None):
        if stage is not None:
            raise IndexOutOfRange(f"dense QP field '{name}' takes no stage index")
        if name not in _SHAPES:
            raise UnknownField(name)
        arr = np.array(value, dtype=int if name in _INT else float)
        shp = _SHAPES[name](self)
        if arr.shape != shp:
            raise DimensionMismatch(f"field '{name}': expected shape {shp}, got {arr.shape}")
        self._data[name] = arr
        self._rev += 1

    def get_field(self, name, stage=None):
        if stage is not None:
            raise IndexOutOfRange(f"dense QP field '{name}' takes no stage index")
        if name not in _SHAPES:
            raise UnknownField(name)
        return self._data[name].copy()


def dense_to_ocp(dq: DenseQp) -> OcpQp:
    """The N = 0, nx = 0 optimal-control form of a dense QP without equalities."""
    if dq.ne:
        raise NotImplementedError(
            "dense QPs with equality constraints (ne > 0: kkt_dense Schur / null-space "
            "paths) are not provided; full condensing always yields ne = 0")
    q = OcpQp(OcpQpDim(0, [0], [dq.nv], [dq.nb], [dq.ng], [dq.ns]))
    for f, g in _TO_OCP.items():
        q.set_field(g, 0, dq._data[f])
    return q


def ocp_to_dense(q) -> DenseQp:
    """Inverse of :func:`dense_to_ocp` (an OcpQp with N = 0 and nx = 0)."""
    d = q.dim
    if d.N != 0 or int(d.nx[0]) != 0:
        raise DimensionMismatch("expected a single-stage OCP-QP without states")
    dq = DenseQp(int(d.nu[0]), 0, int(d.nb[0]), int(d.ng[0]), int(d.ns[0]))
    for f, g in _TO_OCP.items():
        dq.set_field(f, q.get_field(g, 0))
    return dq


class DenseLayout:
    """Flat layout of a dense QP without soft rows (view.DenseView,
    view.py:295-336): y = v, pi over the ne equality rows, lam / t over
    [lower nb+ng | upper nb+ng]."""

    kind = "dense"

    def __init__(self, nv, ne, nb, ng):
        self.nv, self.ne, self.nb, self.ng = int(nv), int(ne), int(nb), int(ng)
        self.ns_tot = 0
        self.ny = self.nv
        self.nc = 2 * (self.nb + self.ng)
        self.N = 0
        self.u_off, self.x_off, self.pi_off, self.c_off, self.s_off = [0], [self.nv], [], [0], [0]


_DENSE_PLANS = {}


def _dense_plan(nv, ne, nb, ng, idxb, B, method, dev):
    import ctypes

    from . import _native as nat

    key = (nv, ne, nb, ng, tuple(int(i) for i in idxb), B, method, dev)
    h = _DENSE_PLANS.get(key)
    if h is None:
        import torch

        ib = np.ascontiguousarray(np.asarray(idxb, dtype=np.int32))
        dim = nat.OcpDenseDimC(nv, ne, nb, ng, 0, ib.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        hp = ctypes.c_void_p()
        with torch.cuda.device(dev):
            nat.check(nat.lib().ocpqp_dense_plan_create(ctypes.byref(dim), B, method,
                                                        ctypes.byref(hp)))
        h = hp
        while len(_DENSE_PLANS) >= 8:
            nat.lib().ocpqp_dense_plan_destroy(_DENSE_PLANS.pop(next(iter(_DENSE_PLANS))))
        _DENSE_PLANS[key] = h
    return h


def solve_dense_qp_batch(qps, arg=None, device="cuda"):
    """Batched solve of dense QPs with equality constraints (identical
    nv, ne, nb, ng, idxb) on the GPU: one kernel launch, one CTA per QP.

    Returns a dict of device tensors (y = v, pi, lam, t, status, iters, res,
    flops, trace) in the dense flat layout (:class:`DenseLayout`)."""
    import ctypes

    import torch

    from . import _native as nat
    from .ipm import IpmArg
    from .solver import _check_arg

    arg = _check_arg(arg or IpmArg())
    qps = list(qps)
    q0 = qps[0]
    if any(q.ns for q in qps):
        raise NotImplementedError("dense QPs with equality constraints and soft rows are not provided")
    for q in qps:
        if (q.nv, q.ne, q.nb, q.ng) != (q0.nv, q0.ne, q0.nb, q0.ng) or not np.array_equal(
                q._data["idxb"], q0._data["idxb"]):
            raise DimensionMismatch("a dense batch needs identical nv, ne, nb, ng and idxb")
    if (arg.itref_corr_max > 0 or arg.use_qr_fallback or arg.use_qr_always or arg.abs_form
            or not arg.pred_corr):
        raise NotImplementedError(
            "dense QPs with equality constraints run the speed-mode loop (mode_preset('speed')); "
            "refinement, QR and the absolute form are not provided on this path")
    method = {"schur": 0, "null_space": 1}.get(arg.kkt_method)
    if method is None:
        raise ValueError(f"unknown kkt_method '{arg.kkt_method}'")
    B = len(qps)
    dev = torch.device(device)
    dev_i = dev.index if dev.index is not None else torch.cuda.current_device()
    f64 = dict(dtype=torch.float64, device=dev)
    fields = {}
    for f in nat.DENSE_FIELDS:
        fields[f] = torch.as_tensor(np.stack([np.asarray(q._data[f], dtype=float).reshape(-1)
                                              for q in qps]), **f64).contiguous()
    lay = DenseLayout(q0.nv, q0.ne, q0.nb, q0.ng)
    out = dict(y=torch.empty((B, lay.ny), **f64), pi=torch.empty((B, lay.ne), **f64),
               lam=torch.empty((B, lay.nc), **f64), t=torch.empty((B, lay.nc), **f64),
               status=torch.empty(B, dtype=torch.int32, device=dev),
               iters=torch.empty(B, dtype=torch.int32, device=dev),
               res=torch.empty((B, 5), **f64), flops=torch.empty(B, dtype=torch.int64, device=dev),
               trace=torch.zeros((B, max(1, arg.iter_max), 8), **f64))
    h = _dense_plan(q0.nv, q0.ne, q0.nb, q0.ng, q0._data["idxb"], B, method, dev_i)
    dc = nat.OcpDenseDataC()
    for i, f in enumerate(nat.DENSE_FIELDS):
        t = fields[f]
        setattr(dc, f, t.data_ptr() if t.numel() else None)
        dc.batch_stride[i] = t.shape[1] if t.numel() else 0
    from dataclasses import replace

    carg = nat.arg_to_c(replace(arg, warm_start="none"))
    it = nat.OcpIterC(out["y"].data_ptr(), out["pi"].data_ptr(), out["lam"].data_ptr(),
                      out["t"].data_ptr())
    st = nat.OcpStatsC(out["status"].data_ptr(), out["iters"].data_ptr(), out["res"].data_ptr(),
                       out["flops"].data_ptr(), out["trace"].data_ptr())
    s = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev_i):
        nat.check(nat.lib().ocpqp_dense_solve(h, ctypes.byref(dc), ctypes.byref(carg),
                                              float(arg.reg_dual), ctypes.byref(it),
                                              ctypes.byref(st), ctypes.c_void_p(s.cuda_stream)))
    out["layout"] = lay
    return out


def _dense_residuals(qp, v, pi, lam, t):
    """Final residuals at the returned point (view.py:272-288, DenseView)."""
    from .layout import QpResiduals

    d = qp._data
    m = qp.nb + qp.ng
    lo = np.concatenate([d["lb"], d["lg"]])
    up = np.concatenate([d["ub"], d["ug"]])
    act = np.concatenate([(d["maskl"] != 0) & np.isfinite(lo), (d["masku"] != 0) & np.isfinite(up)])
    dvec = np.concatenate([lo, -up])
    rows = np.concatenate([v[d["idxb"]], d["C"] @ v]) if m else np.zeros(0)
    cy = np.concatenate([rows, -rows])
    lam_a = np.where(act, lam, 0.0)
    t_a = np.where(act, t, 0.0)
    coeff = lam_a[:m] - lam_a[m:]
    ct = np.zeros(qp.nv)
    np.add.at(ct, d["idxb"], coeff[:qp.nb])
    ct += d["C"].T @ coeff[qp.nb:]
    r_g = d["H"] @ v + d["g"] - d["A"].T @ pi - ct
    r_b = -(d["A"] @ v) + d["b"]
    r_d = np.where(act, -cy + np.where(act, dvec, 0.0) + t_a, 0.0)
    r_m = np.where(act, lam_a * t_a, 0.0)
    n_act = int(act.sum())
    mu = float(lam_a @ t_a) / n_act if n_act else 0.0
    nrm = lambda x: float(np.max(np.abs(x))) if x.size else 0.0  # noqa: E731
    return QpResiduals(r_g=r_g, r_b=r_b, r_d=r_d, r_m=r_m, res_g=nrm(r_g), res_b=nrm(r_b),
                       res_d=nrm(r_d), res_m=nrm(r_m), mu=mu)


def solve_dense_qp(qp: DenseQp, arg=None, guess=None):
    """Solve one dense QP (drop-in for mpcqp.solve_dense_qp, solver.py:98-100).

    Returns a SolveReport whose solution has the dense layout: ``y = [v, sl,
    su]`` (``.v``, ``.sl_all``, ``.su_all``), ``lam`` / ``t`` over
    ``[lower nb+ng | upper nb+ng | lower ns | upper ns]``.
    """
    from .solver import solve_ocp_qp

    if not isinstance(qp, DenseQp):
        raise TypeError("solve_dense_qp expects a DenseQp")
    if not qp.ne:
        return solve_ocp_qp(dense_to_ocp(qp), arg, guess)
    if guess is not None and arg is not None and arg.warm_start != "none":
        raise NotImplementedError("warm starts of dense QPs with equality constraints are not provided")
    from .ipm import STATUS_CODES, IterRecord, SolverStats
    from .layout import QpSolution
    from .solver import SolveReport

    out = solve_dense_qp_batch([qp], arg)
    h = {k: v.cpu().numpy() for k, v in out.items() if k != "layout"}
    code = int(h["status"][0])
    it = int(h["iters"][0])
    sol = QpSolution(out["layout"], h["y"][0].copy(), h["pi"][0].copy(), h["lam"][0].copy(),
                     h["t"][0].copy())
    trace = [IterRecord(k, *[float(x) for x in h["trace"][0, k]]) for k in range(it)]
    r = h["res"][0]
    stats = SolverStats(status=STATUS_CODES[code], iterations=it, res_g=float(r[0]),
                        res_b=float(r[1]), res_d=float(r[2]), res_m=float(r[3]), mu=float(r[4]),
                        flops=int(h["flops"][0]), trace=trace)
    res = _dense_residuals(qp, sol.y, sol.pi, sol.lam, sol.t)
    return SolveReport(solution=sol, stats=stats, residuals=res)
