"""Packed batch of structurally identical OCP-QPs (the layout the kernels read).

One array per catalog field, shape ``[Bf, L_f]`` where ``L_f`` is the packed
length of the field over all stages (layout.FIELD_ORDER, canonical order of
include/ocpqp_b200.h) and ``Bf`` is either the batch size or 1 (one copy
broadcast to every QP, e.g. the shared plant of the mass-spring benchmarks).
A missing field means the reference's zero-initialised default
(qp_data.py:221-245).  ``idxb``/``idxs`` are structural and shared.

``from_qps`` packs a list of reference-style ``OcpQp`` objects (the drop-in
path); the benchmark generators fill the arrays directly.
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch
from .layout import FIELD_ORDER, OcpLayout, field_shape
from .qp_data import OcpQp, OcpQpDim

__all__ = ["OcpQpBatch"]

_DYN = ("A", "B", "b")


class OcpQpBatch:
    """Struct-of-arrays batch; fields are numpy arrays or torch tensors."""

    def __init__(self, dim: OcpQpDim, batch: int, idxb=None, idxs=None, fields=None):
        self.dim = dim
        self.B = int(batch)
        self.layout = OcpLayout(dim)
        d = dim
        if idxb is None:
            idxb = [np.arange(d.nb[n]) for n in range(d.N + 1)]
        if idxs is None:
            idxs = [np.arange(d.ns[n]) for n in range(d.N + 1)]
        self.idxb = [np.asarray(a, dtype=np.int32).reshape(-1) for a in idxb]
        self.idxs = [np.asarray(a, dtype=np.int32).reshape(-1) for a in idxs]
        for n in range(d.N + 1):
            if self.idxb[n].shape[0] != d.nb[n] or self.idxs[n].shape[0] != d.ns[n]:
                raise DimensionMismatch(f"stage {n}: idxb/idxs length mismatch")
        self.fields = {}
        for name, arr in (fields or {}).items():
            self.set_packed(name, arr)

    # -- packed storage -------------------------------------------------------
    def set_packed(self, name, arr):
        if name not in FIELD_ORDER:
            raise KeyError(name)
        L = self.layout.field_len[name]
        if arr is None:
            self.fields.pop(name, None)
            return
        if hasattr(arr, "ndim") and arr.ndim == 1:
            arr = arr.reshape(1, -1)
        if arr.shape[-1] != L or arr.shape[0] not in (1, self.B):
            raise DimensionMismatch(
                f"field {name}: expected [1 or {self.B}, {L}], got {tuple(arr.shape)}")
        self.fields[name] = arr

    def alloc(self, name, per_qp: bool, fill=None):
        """Allocate (numpy) storage for a field and return it."""
        L = self.layout.field_len[name]
        rows = self.B if per_qp else 1
        if fill is None:
            fill = default_fill(name)
        arr = np.full((rows, L), fill, dtype=np.float64)
        self.fields[name] = arr
        return arr

    def stage_view(self, name, n):
        """View ``[Bf, *shape]`` of stage n of a (numpy) packed field."""
        arr = self.fields[name]
        shp = field_shape(name, self.dim, n)
        sl = self.layout.stage_slice(name, n)
        return arr[:, sl].reshape((arr.shape[0],) + tuple(shp))

    def idxb_concat(self):
        return (np.concatenate(self.idxb) if self.idxb else np.zeros(0)).astype(np.int32)

    def idxs_concat(self):
        return (np.concatenate(self.idxs) if self.idxs else np.zeros(0)).astype(np.int32)

    def structure_key(self):
        # idxb / idxs are fixed at construction; the key is cached
        key = getattr(self, "_skey", None)
        if key is None:
            key = (self.dim.key(), tuple(self.idxb_concat().tolist()),
                   tuple(self.idxs_concat().tolist()))
            self._skey = key
        return key

    # -- conversions -----------------------------------------------------------
    def to(self, device):
        """Copy with every field as a contiguous float64 torch tensor on ``device``."""
        import torch

        out = OcpQpBatch(self.dim, self.B, self.idxb, self.idxs)
        for name, arr in self.fields.items():
            if isinstance(arr, np.ndarray):
                t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
            else:
                t = arr
            out.fields[name] = t.to(device=device, dtype=torch.float64).contiguous()
        return out

    def numpy(self):
        """Copy with every field as a numpy array (host)."""
        out = OcpQpBatch(self.dim, self.B, self.idxb, self.idxs)
        for name, arr in self.fields.items():
            if not isinstance(arr, np.ndarray):
                arr = arr.detach().cpu().numpy()
            out.fields[name] = np.ascontiguousarray(arr, dtype=np.float64)
        return out

    def pin_memory(self):
        """Copy with every field as a pinned-host torch tensor (for timed H2D)."""
        import torch

        out = OcpQpBatch(self.dim, self.B, self.idxb, self.idxs)
        for name, arr in self.fields.items():
            t = torch.from_numpy(np.ascontiguousarray(arr)) if isinstance(arr, np.ndarray) else arr
            out.fields[name] = t.to(torch.float64).contiguous().pin_memory()
        return out

    def select(self, indices):
        """Sub-batch of the given QP indices (host numpy batch)."""
        idx = np.asarray(indices, dtype=int)
        src = self.numpy()
        out = OcpQpBatch(self.dim, len(idx), self.idxb, self.idxs)
        for name, arr in src.fields.items():
            out.fields[name] = arr if arr.shape[0] == 1 else np.ascontiguousarray(arr[idx])
        return out

    @classmethod
    def from_qps(cls, qps):
        """Pack reference-style OcpQp objects sharing dims, idxb and idxs."""
        qps = list(qps)
        if not qps:
            raise ValueError("empty QP list")
        q0 = qps[0]
        if not isinstance(q0, OcpQp) and not hasattr(q0, "_stages"):
            raise TypeError("expected OcpQp objects")
        dim = q0.dim
        d = dim
        idxb = [np.asarray(q0._stages[n]["idxb"]) for n in range(d.N + 1)]
        idxs = [np.asarray(q0._stages[n]["idxs"]) for n in range(d.N + 1)]
        key = _dim_key(dim)
        for q in qps[1:]:
            if _dim_key(q.dim) != key:
                raise DimensionMismatch("all QPs of a batch must share the dimensions")
            for n in range(d.N + 1):
                if (not np.array_equal(q._stages[n]["idxb"], idxb[n])
                        or not np.array_equal(q._stages[n]["idxs"], idxs[n])):
                    raise DimensionMismatch("all QPs of a batch must share idxb / idxs")
        out = cls(dim, len(qps), idxb, idxs)
        lay = out.layout
        for name in FIELD_ORDER:
            L = lay.field_len[name]
            if L == 0:
                continue
            arr = np.empty((len(qps), L))
            for i, q in enumerate(qps):
                for n in range(d.N + 1):
                    if name in _DYN:
                        if n == d.N:
                            continue
                        src = q._dyn[n][name]
                    else:
                        src = q._stages[n][name]
                    arr[i, lay.stage_slice(name, n)] = np.asarray(src, dtype=float).reshape(-1)
            if len(qps) > 1 and np.all(arr == arr[:1]) and not np.any(np.isnan(arr)):
                arr = np.ascontiguousarray(arr[:1])
            out.fields[name] = arr
        return out

    def qp(self, i) -> OcpQp:
        """Unpack QP ``i`` into an OcpQp (host)."""
        src = self.numpy()
        d = self.dim
        q = OcpQp(d)
        lay = self.layout
        for n in range(d.N + 1):
            q.set_field("idxb", n, self.idxb[n].astype(int))
            q.set_field("idxs", n, self.idxs[n].astype(int))
        for name, arr in src.fields.items():
            row = arr[0 if arr.shape[0] == 1 else i]
            for n in range(d.N + 1):
                if name in _DYN and n == d.N:
                    continue
                shp = field_shape(name, d, n)
                q.set_field(name, n, row[lay.stage_slice(name, n)].reshape(shp))
        return q


def _dim_key(dim):
    return (dim.N, tuple(map(int, dim.nx)), tuple(map(int, dim.nu)), tuple(map(int, dim.nb)),
            tuple(map(int, dim.ng)), tuple(map(int, dim.ns)))


def default_fill(name):
    if name in ("lb", "lg"):
        return -np.inf
    if name in ("ub", "ug"):
        return np.inf
    if name in ("maskl", "masku"):
        return 1.0
    return 0.0
