"""Text interchange format of optimal-control QPs (reference qp_io.py, version 1).

Same file layout as the reference's ``qp_write`` / ``qp_read``
(/root/reference/pkg/src/mpcqp/qp_io.py:1-31, 197-308) for the ``ocp`` kind:
a ``mpcqp_qp 1 ocp`` header, ``N`` and the per-stage count lines, then one
``stage n`` section per stage with the catalog fields in a fixed order (cost,
bounds, general rows, soft rows, masks) followed by the dynamics blocks
``A B b`` for n < N.  A field is its name on one line and its values below:
one line per matrix row, one line for a vector or index set, no line for an
empty matrix.  Floats are written with ``repr`` (shortest round trip, ``inf``
/ ``-inf``), so a write followed by a read is bit-exact and a file written
here is byte-identical to the reference's for the same QP.

Reading is strict: a wrong field name, count or number, a truncated file or
trailing content raises :class:`ParseError` with the line number; another
format version raises :class:`VersionMismatch`.  The ``dense`` and ``tree``
kinds are outside this package (the GPU path solves OCP QPs) and are
rejected with ParseError.
"""

from __future__ import annotations

import numpy as np

from .errors import ParseError, VersionMismatch
from .qp_data import OcpQp, OcpQpDim

__all__ = ["qp_read", "qp_write", "qp_dumps", "qp_loads"]

MAGIC = "mpcqp_qp"
VERSION = 1
STAGE_FIELDS = ("Q", "S", "R", "q", "r", "idxb", "lb", "ub", "C", "D", "lg", "ug",
                "idxs", "Zl", "Zu", "zl", "zu", "sl_lb", "su_lb", "maskl", "masku")
DYN_FIELDS = ("A", "B", "b")
INDEX_FIELDS = ("idxb", "idxs")


def _num(x):
    return repr(float(x))


def _emit(lines, name, value):
    lines.append(name)
    a = np.asarray(value)
    if a.ndim == 1:
        if name in INDEX_FIELDS:
            lines.append(" ".join(str(int(v)) for v in a))
        else:
            lines.append(" ".join(_num(v) for v in a))
    else:
        lines.extend(" ".join(_num(v) for v in row) for row in a)


def _stage_shape(name, d, n):
    nx, nu, nb, ng, ns = d.nx[n], d.nu[n], d.nb[n], d.ng[n], d.ns[n]
    return {"Q": (nx, nx), "S": (nu, nx), "R": (nu, nu), "q": (nx,), "r": (nu,),
            "idxb": (nb,), "lb": (nb,), "ub": (nb,), "C": (ng, nx), "D": (ng, nu),
            "lg": (ng,), "ug": (ng,), "idxs": (ns,), "Zl": (ns,), "Zu": (ns,), "zl": (ns,),
            "zu": (ns,), "sl_lb": (ns,), "su_lb": (ns,), "maskl": (nb + ng,),
            "masku": (nb + ng,)}[name]


def qp_dumps(qp):
    """The file text of an OcpQp."""
    if not isinstance(qp, OcpQp):
        raise TypeError(f"not an OCP QP: {type(qp)!r}")
    d = qp.dim
    lines = [f"{MAGIC} {VERSION} ocp", f"N {d.N}"]
    for key in ("nx", "nu", "nb", "ng", "ns"):
        lines.append(" ".join([key] + [str(int(v)) for v in getattr(d, key)]))
    for n in range(d.N + 1):
        lines.append(f"stage {n}")
        for name in STAGE_FIELDS:
            _emit(lines, name, qp.get_field(name, n))
        if n < d.N:
            for name in DYN_FIELDS:
                _emit(lines, name, qp.get_field(name, n))
    return "\n".join(lines) + "\n"


def qp_write(path, qp):
    """Write ``qp`` to ``path`` (overwrites)."""
    text = qp_dumps(qp)
    with open(path, "w") as fh:
        fh.write(text)


class _Lines:
    """Line cursor with 1-based error positions."""

    def __init__(self, text):
        self.lines = text.splitlines()
        self.i = 0

    def take(self):
        if self.i >= len(self.lines):
            raise ParseError("unexpected end of file", line=len(self.lines))
        self.i += 1
        return self.lines[self.i - 1]

    def token(self, tok):
        got = self.take().strip()
        if got != tok:
            raise ParseError(f"expected field '{tok}', found '{got}'", line=self.i)

    def counts(self, key, k):
        parts = self.take().split()
        if not parts or parts[0] != key:
            raise ParseError(f"expected '{key}' line, found '{' '.join(parts)}'", line=self.i)
        if len(parts) != k + 1:
            raise ParseError(f"'{key}' expects {k} integers, found {len(parts) - 1}",
                             line=self.i)
        try:
            return [int(t) for t in parts[1:]]
        except ValueError as exc:
            raise ParseError(f"bad integer in '{key}' line: {exc}", line=self.i)

    def values(self, k, cast):
        parts = self.take().split()
        if len(parts) != k:
            what = "integers" if cast is int else "numbers"
            raise ParseError(f"expected {k} {what}, found {len(parts)}", line=self.i)
        try:
            return [cast(t) for t in parts]
        except ValueError as exc:
            raise ParseError(f"bad {'integer' if cast is int else 'number'}: {exc}",
                             line=self.i)

    def field(self, name, shape):
        self.token(name)
        if name in INDEX_FIELDS:
            return np.array(self.values(shape[0], int), dtype=int)
        if len(shape) == 1:
            return np.array(self.values(shape[0], float))
        rows, cols = shape
        return np.array([self.values(cols, float) for _ in range(rows)],
                        dtype=float).reshape(rows, cols)

    def end(self):
        for j in range(self.i, len(self.lines)):
            if self.lines[j].strip():
                raise ParseError("trailing content", line=j + 1)


def qp_loads(text):
    """Parse the file text of an OCP QP."""
    cur = _Lines(text)
    head = cur.take().split()
    if len(head) != 3 or head[0] != MAGIC:
        raise ParseError("not a QP file (bad magic line)", line=1)
    if head[1] != str(VERSION):
        raise VersionMismatch(f"unsupported format version '{head[1]}'", line=1)
    if head[2] != "ocp":
        if head[2] in ("dense", "tree"):
            raise ParseError(f"QP kind '{head[2]}' is not supported by this package "
                             "(optimal-control QPs only)", line=1)
        raise ParseError(f"unknown QP kind '{head[2]}'", line=1)
    (N,) = cur.counts("N", 1)
    dims = {k: cur.counts(k, N + 1) for k in ("nx", "nu", "nb", "ng", "ns")}
    d = OcpQpDim(N, **dims)
    qp = OcpQp(d)
    for n in range(N + 1):
        cur.token(f"stage {n}")
        for name in STAGE_FIELDS:
            qp.set_field(name, n, cur.field(name, _stage_shape(name, d, n)))
        if n < N:
            qp.set_field("A", n, cur.field("A", (d.nx[n + 1], d.nx[n])))
            qp.set_field("B", n, cur.field("B", (d.nx[n + 1], d.nu[n])))
            qp.set_field("b", n, cur.field("b", (d.nx[n + 1],)))
    cur.end()
    return qp


def qp_read(path):
    """Read an OCP QP file."""
    with open(path) as fh:
        return qp_loads(fh.read())
