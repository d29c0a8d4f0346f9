"""Dense QP type and its solve (reference qp_data.DenseQp, qp_data.py:426-500;
solver.solve_dense_qp, solver.py:98-100).

A dense QP without equality constraints (ne = 0, the form full condensing
produces, condensing.py:297) is the single-stage optimal-control QP with
N = 0, nx = 0, nu = nv: H -> R, g -> r, C -> D, the box / general / soft rows
unchanged.  On that form the reference's dense backend (kkt_dense.py:117-256:
Hred = H + C' diag(gamma) C, Cholesky, dv = -Hred^-1 rhat) and its Riccati
backend at N = 0 perform the same operations in the same order -- same
iterates, same iteration counts and the same counted flops (checked against
the reference in tests/golden/fcond.npz) -- so the dense QP is solved by the
same fused sm_100a kernels as every OCP-QP.  Dense QPs with equality
constraints (the Schur / null-space paths, kkt_dense.py:166-185) are not
provided (NotImplementedError).
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch, IndexOutOfRange, InvalidDim, UnknownField
from .qp_data import OcpQp, OcpQpDim

__all__ = ["DenseQp", "dense_to_ocp", "ocp_to_dense", "solve_dense_qp"]

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


def solve_dense_qp(qp: DenseQp, arg=None, guess=None):
    """Solve one dense QP (drop-in for mpcqp.solve_dense_qp, solver.py:98-100).

    Returns a SolveReport whose solution has the dense layout: ``y = [v, sl,
    su]`` (``.v``, ``.sl_all``, ``.su_all``), ``lam`` / ``t`` over
    ``[lower nb+ng | upper nb+ng | lower ns | upper ns]``.
    """
    from .solver import solve_ocp_qp

    if not isinstance(qp, DenseQp):
        raise TypeError("solve_dense_qp expects a DenseQp")
    return solve_ocp_qp(dense_to_ocp(qp), arg, guess)
