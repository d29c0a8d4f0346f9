"""OCP-QP containers of the drop-in API: ``OcpQpDim``, ``OcpQp``, ``validate``.

Behavioural mirror of the reference's optimal-control QP container
(mpcqp/qp_data.py:65-111 ``OcpQpDim``, :221-313 stage catalog and accessors,
:316-364 ``OcpQp``, :509-634 ``validate``):

* stages 0..N carry the cost ``1/2 [u;x]'[R S; S' Q][u;x] + [r;q]'[u;x]``,
  box rows ``lb <= w[idxb] <= ub`` on ``w = (u, x)`` (inputs first), general
  rows ``lg <= D u + C x <= ug``, soft-row data and per-side masks;
* dynamics blocks 0..N-1 carry ``x[n+1] = A x[n] + B u[n] + b``;
* freshly built problems are zero with infinite bounds, all-one masks,
  ``idxb = arange(nb)`` and ``idxs = arange(ns)``;
* ``set_field``/``get_field`` check shapes and return copies; the virtual
  fields ``lbu/ubu/lbx/ubx`` address the input/state subsets of lb/ub.

Storage is one dict per stage, the same shape contract as the reference; the
batch packer (batch.py) reads it directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch, IndexOutOfRange, InvalidDim, UnknownField

__all__ = ["OcpQpDim", "OcpQp", "Violation", "validate", "errors_only",
           "STAGE_FIELDS", "DYN_FIELDS", "VIRTUAL_FIELDS"]


def _as_dims(values, name, count):
    if values is None:
        values = [0] * count
    arr = np.asarray(values, dtype=int)
    if arr.ndim != 1:
        raise InvalidDim(f"{name} must be a 1-d integer sequence")
    if np.any(arr < 0):
        raise InvalidDim(f"{name} entries must be nonnegative")
    if arr.shape[0] != count:
        raise InvalidDim(f"{name} must have N+1 = {count} entries")
    return arr


@dataclass(frozen=True)
class OcpQpDim:
    """Per-stage sizes nx, nu, nb, ng, ns of an OCP-QP with horizon N."""

    N: int
    nx: np.ndarray
    nu: np.ndarray
    nb: np.ndarray
    ng: np.ndarray
    ns: np.ndarray

    def __init__(self, N, nx, nu, nb=None, ng=None, ns=None):
        if N < 0:
            raise InvalidDim("horizon N must be >= 0")
        N = int(N)
        count = N + 1
        object.__setattr__(self, "N", N)
        for name, val in (("nx", nx), ("nu", nu), ("nb", nb), ("ng", ng), ("ns", ns)):
            object.__setattr__(self, name, _as_dims(val, name, count))
        for n in range(count):
            nw = self.nu[n] + self.nx[n]
            if self.nb[n] > nw:
                raise InvalidDim(
                    f"stage {n}: nb = {self.nb[n]} exceeds nu + nx = {nw}")
            if self.ns[n] > self.nb[n] + self.ng[n]:
                raise InvalidDim(
                    f"stage {n}: ns = {self.ns[n]} exceeds nb + ng = "
                    f"{self.nb[n] + self.ng[n]}")

    def key(self):
        """Hashable structural key (used to group QPs into one batch)."""
        return (self.N, tuple(self.nx), tuple(self.nu), tuple(self.nb),
                tuple(self.ng), tuple(self.ns))


# field -> (shape(dim, n), dtype); dynamics fields are indexed 0..N-1
STAGE_FIELDS = {
    "Q": (lambda d, n: (d.nx[n], d.nx[n]), float),
    "S": (lambda d, n: (d.nu[n], d.nx[n]), float),
    "R": (lambda d, n: (d.nu[n], d.nu[n]), float),
    "q": (lambda d, n: (d.nx[n],), float),
    "r": (lambda d, n: (d.nu[n],), float),
    "idxb": (lambda d, n: (d.nb[n],), int),
    "lb": (lambda d, n: (d.nb[n],), float),
    "ub": (lambda d, n: (d.nb[n],), float),
    "C": (lambda d, n: (d.ng[n], d.nx[n]), float),
    "D": (lambda d, n: (d.ng[n], d.nu[n]), float),
    "lg": (lambda d, n: (d.ng[n],), float),
    "ug": (lambda d, n: (d.ng[n],), float),
    "idxs": (lambda d, n: (d.ns[n],), int),
    "Zl": (lambda d, n: (d.ns[n],), float),
    "Zu": (lambda d, n: (d.ns[n],), float),
    "zl": (lambda d, n: (d.ns[n],), float),
    "zu": (lambda d, n: (d.ns[n],), float),
    "sl_lb": (lambda d, n: (d.ns[n],), float),
    "su_lb": (lambda d, n: (d.ns[n],), float),
    "maskl": (lambda d, n: (d.nb[n] + d.ng[n],), float),
    "masku": (lambda d, n: (d.nb[n] + d.ng[n],), float),
}
DYN_FIELDS = {
    "A": (lambda d, n: (d.nx[n + 1], d.nx[n]), float),
    "B": (lambda d, n: (d.nx[n + 1], d.nu[n]), float),
    "b": (lambda d, n: (d.nx[n + 1],), float),
}
VIRTUAL_FIELDS = ("lbu", "ubu", "lbx", "ubx")


def _default_stage(nx, nu, nb, ng, ns):
    """Zero-initialised stage (qp_data.py:221-245)."""
    return {
        "Q": np.zeros((nx, nx)), "S": np.zeros((nu, nx)), "R": np.zeros((nu, nu)),
        "q": np.zeros(nx), "r": np.zeros(nu),
        "idxb": np.arange(nb, dtype=int),
        "lb": np.full(nb, -np.inf), "ub": np.full(nb, np.inf),
        "C": np.zeros((ng, nx)), "D": np.zeros((ng, nu)),
        "lg": np.full(ng, -np.inf), "ug": np.full(ng, np.inf),
        "idxs": np.arange(ns, dtype=int),
        "Zl": np.zeros(ns), "Zu": np.zeros(ns), "zl": np.zeros(ns), "zu": np.zeros(ns),
        "sl_lb": np.zeros(ns), "su_lb": np.zeros(ns),
        "maskl": np.ones(nb + ng), "masku": np.ones(nb + ng),
    }


def _checked(name, value, shape, dtype):
    arr = np.array(value, dtype=dtype)
    if arr.shape != tuple(shape):
        raise DimensionMismatch(
            f"field '{name}': expected shape {tuple(shape)}, got {arr.shape}")
    return arr


class OcpQp:
    """Optimal-control QP over stages 0..N, zero-initialised."""

    kind = "ocp"

    def __init__(self, dim: OcpQpDim):
        if not isinstance(dim, OcpQpDim):
            raise InvalidDim("OcpQp requires an OcpQpDim")
        self.dim = dim
        d = dim
        self._stages = [
            _default_stage(d.nx[n], d.nu[n], d.nb[n], d.ng[n], d.ns[n])
            for n in range(d.N + 1)
        ]
        self._dyn = [
            {"A": np.zeros((d.nx[n + 1], d.nx[n])),
             "B": np.zeros((d.nx[n + 1], d.nu[n])),
             "b": np.zeros(d.nx[n + 1])}
            for n in range(d.N)
        ]
        self._rev = 0

    # -- catalog ------------------------------------------------------------
    def field_names(self):
        return sorted(set(STAGE_FIELDS) | set(DYN_FIELDS) | set(VIRTUAL_FIELDS))

    def _stage_check(self, name, n, dyn):
        hi = self.dim.N - 1 if dyn else self.dim.N
        if not 0 <= n <= hi:
            raise IndexOutOfRange(f"field '{name}': stage {n} outside 0..{hi}")

    def _input_rows(self, n):
        return self._stages[n]["idxb"] < self.dim.nu[n]

    def set_field(self, name, stage, value):
        """Store ``value`` for field ``name`` at ``stage``."""
        if name in VIRTUAL_FIELDS:
            self._stage_check(name, stage, False)
            rows = self._input_rows(stage)
            if name.endswith("x"):
                rows = ~rows
            dst = "lb" if name[0] == "l" else "ub"
            arr = _checked(name, value, (int(rows.sum()),), float)
            new = self._stages[stage][dst].copy()
            new[rows] = arr
            self._stages[stage][dst] = new
            self._rev += 1
            return
        if name in STAGE_FIELDS:
            shape, dtype = STAGE_FIELDS[name]
            self._stage_check(name, stage, False)
            self._stages[stage][name] = _checked(name, value, shape(self.dim, stage), dtype)
        elif name in DYN_FIELDS:
            shape, dtype = DYN_FIELDS[name]
            self._stage_check(name, stage, True)
            self._dyn[stage][name] = _checked(name, value, shape(self.dim, stage), dtype)
        else:
            raise UnknownField(name)
        self._rev += 1

    def get_field(self, name, stage):
        """Copy of the stored values of field ``name`` at ``stage``."""
        if name in VIRTUAL_FIELDS:
            self._stage_check(name, stage, False)
            rows = self._input_rows(stage)
            if name.endswith("x"):
                rows = ~rows
            src = "lb" if name[0] == "l" else "ub"
            return self._stages[stage][src][rows].copy()
        if name in STAGE_FIELDS:
            self._stage_check(name, stage, False)
            return self._stages[stage][name].copy()
        if name in DYN_FIELDS:
            self._stage_check(name, stage, True)
            return self._dyn[stage][name].copy()
        raise UnknownField(name)


# ----------------------------------------------------------------------------
# validation (qp_data.py:509-634)
# ----------------------------------------------------------------------------
@dataclass
class Violation:
    """One diagnostic of :func:`validate`; severity 'error' or 'warning'."""

    field: str
    stage: object
    message: str
    severity: str = "error"

    def __str__(self):
        where = "" if self.stage is None else f" [stage {self.stage}]"
        return f"{self.severity}: {self.field}{where}: {self.message}"


def _check_stage(st, nu, nx, nb, ng, n, out):
    for name in ("Q", "R"):
        M = st[name]
        if M.shape[0]:
            tol = 1e-10 * max(1.0, float(np.max(np.abs(M))))
            if not np.allclose(M, M.T, rtol=0.0, atol=tol):
                out.append(Violation(name, n, "matrix is not symmetric"))
    for name in ("Zl", "Zu"):
        if np.any(st[name] < 0.0):
            out.append(Violation(name, n, "slack penalty diagonal must be >= 0"))
    for name, limit in (("idxb", nu + nx), ("idxs", nb + ng)):
        idx = st[name]
        if idx.size and (np.any(idx < 0) or np.any(idx >= limit)):
            out.append(Violation(name, n, f"entries must lie in [0, {limit})"))
        if idx.size > 1 and np.any(np.diff(idx) <= 0):
            out.append(Violation(name, n, "entries must be strictly increasing"))
    for name in ("maskl", "masku"):
        mk = st[name]
        if mk.size and not np.all((mk == 0.0) | (mk == 1.0)):
            out.append(Violation(name, n, "mask entries must be 0 or 1"))
    lo = np.concatenate([st["lb"], st["lg"]])
    up = np.concatenate([st["ub"], st["ug"]])
    both = (st["maskl"] != 0.0) & (st["masku"] != 0.0)
    crossed = both & np.isfinite(lo) & np.isfinite(up) & (lo > up)
    for i in np.flatnonzero(crossed):
        out.append(Violation("lb/ub" if i < nb else "lg/ug", n,
                             f"row {i}: lower bound exceeds upper bound",
                             severity="warning"))
    if np.any(st["sl_lb"] < 0.0) or np.any(st["su_lb"] < 0.0):
        out.append(Violation("sl_lb/su_lb", n,
                             "negative slack lower bound (allowed, check intent)",
                             severity="warning"))


def validate(qp):
    """Diagnostics for an OCP QP; an empty list means valid."""
    if not isinstance(qp, OcpQp):
        raise TypeError(f"not an OCP QP container: {type(qp)!r}")
    out = []
    d = qp.dim
    for n in range(d.N + 1):
        _check_stage(qp._stages[n], d.nu[n], d.nx[n], d.nb[n], d.ng[n], n, out)
    return out


def errors_only(violations):
    """The blocking (severity 'error') entries of a validate() result."""
    return [v for v in violations if v.severity == "error"]
