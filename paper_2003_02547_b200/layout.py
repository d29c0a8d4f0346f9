"""Flat layout of one OCP-QP and the solution / residual records.

The flat vectors are exactly the reference's (mpcqp/view.py:3-13, OcpView
:337-366): ``y = [v | sl | su]`` with ``v = (u_0, x_0, u_1, x_1, ...)``,
``pi = (pi_0 .. pi_{N-1})`` and per stage ``lam``/``t`` slots
``[lower m | upper m | slack-lower ns | slack-upper ns]`` with ``m = nb + ng``.
The per-field packed lengths/offsets are the canonical batch layout of the C
ABI (include/ocpqp_b200.h): stage-major, matrices row-major, dynamics fields
for stages 0..N-1 only.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch

__all__ = ["FIELD_ORDER", "OcpLayout", "QpSolution", "QpResiduals"]

# field order of the C ABI enum OcpQpField
FIELD_ORDER = ("A", "B", "b", "Q", "S", "R", "q", "r", "lb", "ub", "C", "D", "lg",
               "ug", "Zl", "Zu", "zl", "zu", "sl_lb", "su_lb", "maskl", "masku")
FIELD_INDEX = {name: i for i, name in enumerate(FIELD_ORDER)}


def field_shape(name, dim, n):
    """Per-stage shape of a packed field (empty for dynamics fields at n = N)."""
    nx, nu, nb, ng, ns = (int(dim.nx[n]), int(dim.nu[n]), int(dim.nb[n]),
                          int(dim.ng[n]), int(dim.ns[n]))
    nxn = int(dim.nx[n + 1]) if n < dim.N else 0
    if name in ("A", "B", "b") and n == dim.N:
        return (0,)
    return {
        "A": (nxn, nx), "B": (nxn, nu), "b": (nxn,),
        "Q": (nx, nx), "S": (nu, nx), "R": (nu, nu), "q": (nx,), "r": (nu,),
        "lb": (nb,), "ub": (nb,), "C": (ng, nx), "D": (ng, nu), "lg": (ng,), "ug": (ng,),
        "Zl": (ns,), "Zu": (ns,), "zl": (ns,), "zu": (ns,), "sl_lb": (ns,), "su_lb": (ns,),
        "maskl": (nb + ng,), "masku": (nb + ng,),
    }[name]


class OcpLayout:
    """Offsets of the flat vectors and of the packed fields for one dims record."""

    kind = "ocp"

    def __init__(self, dim):
        self.dim = dim
        d = dim
        N = d.N
        self.N = N
        self.u_off, self.x_off, self.pi_off, self.c_off, self.s_off = [], [], [], [], []
        v = s = c = p = 0
        for n in range(N + 1):
            self.u_off.append(v)
            self.x_off.append(v + int(d.nu[n]))
            self.s_off.append(s)
            self.c_off.append(c)
            v += int(d.nu[n] + d.nx[n])
            s += int(d.ns[n])
            c += 2 * int(d.nb[n] + d.ng[n]) + 2 * int(d.ns[n])
            if n < N:
                self.pi_off.append(p)
                p += int(d.nx[n + 1])
        self.nv, self.ns_tot, self.nc, self.ne = v, s, c, p
        self.ny = v + 2 * s
        # packed field offsets
        self.field_len = {}
        self.field_off = {}
        for name in FIELD_ORDER:
            offs, tot = [], 0
            for n in range(N + 1):
                offs.append(tot)
                tot += int(np.prod(field_shape(name, d, n)))
            self.field_off[name] = offs
            self.field_len[name] = tot

    def stage_nc(self, n):
        d = self.dim
        return 2 * int(d.nb[n] + d.ng[n]) + 2 * int(d.ns[n])

    def m(self, n):
        return int(self.dim.nb[n] + self.dim.ng[n])

    def stage_slice(self, name, n):
        off = self.field_off[name][n]
        size = int(np.prod(field_shape(name, self.dim, n)))
        return slice(off, off + size)


class QpSolution:
    """Primal-dual point of one QP; mirrors view.QpSolution (view.py:568-672)."""

    def __init__(self, layout, y=None, pi=None, lam=None, t=None):
        self._layout = layout
        self.y = np.zeros(layout.ny) if y is None else y
        self.pi = np.zeros(layout.ne) if pi is None else pi
        self.lam = np.zeros(layout.nc) if lam is None else lam
        self.t = np.zeros(layout.nc) if t is None else t

    @property
    def kind(self):
        return self._layout.kind

    @property
    def layout(self):
        return self._layout

    @property
    def v(self):
        return self.y[: self._layout.nv]

    @property
    def sl_all(self):
        L = self._layout
        return self.y[L.nv: L.nv + L.ns_tot]

    @property
    def su_all(self):
        return self.y[self._layout.nv + self._layout.ns_tot:]

    def u(self, n):
        L = self._layout
        return self.y[L.u_off[n]: L.u_off[n] + int(L.dim.nu[n])]

    def x(self, n):
        L = self._layout
        return self.y[L.x_off[n]: L.x_off[n] + int(L.dim.nx[n])]

    def sl(self, n):
        L = self._layout
        return self.sl_all[L.s_off[n]: L.s_off[n] + int(L.dim.ns[n])]

    def su(self, n):
        L = self._layout
        return self.su_all[L.s_off[n]: L.s_off[n] + int(L.dim.ns[n])]

    def pi_stage(self, n):
        L = self._layout
        return self.pi[L.pi_off[n]: L.pi_off[n] + int(L.dim.nx[n + 1])]

    def lam_stage(self, n):
        L = self._layout
        return self.lam[L.c_off[n]: L.c_off[n] + L.stage_nc(n)]

    def t_stage(self, n):
        L = self._layout
        return self.t[L.c_off[n]: L.c_off[n] + L.stage_nc(n)]

    def copy(self):
        return QpSolution(self._layout, self.y.copy(), self.pi.copy(),
                          self.lam.copy(), self.t.copy())

    def axpy(self, alpha, step):
        self.y += alpha * step.y
        self.pi += alpha * step.pi
        self.lam += alpha * step.lam
        self.t += alpha * step.t

    def diff(self, other):
        return QpSolution(self._layout, self.y - other.y, self.pi - other.pi,
                          self.lam - other.lam, self.t - other.t)

    def flat(self):
        return np.concatenate([self.y, self.pi, self.lam, self.t])

    @classmethod
    def from_flat(cls, layout, vec):
        ny, ne, nc = layout.ny, layout.ne, layout.nc
        if vec.shape[0] != ny + ne + 2 * nc:
            raise DimensionMismatch("flat vector length does not match the layout")
        return cls(layout, vec[:ny].copy(), vec[ny: ny + ne].copy(),
                   vec[ny + ne: ny + ne + nc].copy(), vec[ny + ne + nc:].copy())

    def isfinite(self):
        return all(bool(np.all(np.isfinite(a))) for a in (self.y, self.pi, self.lam, self.t))


@dataclass
class QpResiduals:
    """KKT residual blocks, their infinity norms and the duality measure."""

    r_g: np.ndarray
    r_b: np.ndarray
    r_d: np.ndarray
    r_m: np.ndarray
    res_g: float
    res_b: float
    res_d: float
    res_m: float
    mu: float

    def max_norm(self):
        return max(self.res_g, self.res_b, self.res_d, self.res_m)

    def isfinite(self):
        return all(np.isfinite(x) for x in (self.res_g, self.res_b, self.res_d, self.res_m))
