"""Batched partial condensing / expansion on the GPU (reference condensing.py:451-619).

``partial_condense_batch(batch, N1)`` turns a batch of OCP-QPs with horizon N
into the batch of block-condensed QPs with horizon ceil(N / N1) (each block of
N1 stages condensed with its initial state kept; the old terminal stage carried
over verbatim), and ``partial_expand_batch`` maps the short-horizon solutions
back to the full horizon (forward state rollout, multiplier routing, costate
recursion for pi).  The routing tables are built once per structure by the C
ABI (ocpqp_pc_create); the arithmetic runs in the CUDA kernels of
csrc/ocpqp_condense.cu.  ``partial_condense`` / ``partial_expand`` are the
reference's single-QP calls.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .batch import OcpQpBatch, default_fill
from .errors import InvalidBlockSize, NativeLibraryError
from .layout import FIELD_ORDER, QpSolution
from .qp_data import OcpQp, OcpQpDim

__all__ = ["PartialCondensingMap", "partial_condense_batch", "partial_expand_batch",
           "partial_condense", "partial_expand"]


def _lib():
    L = nat.lib()
    if not getattr(L, "_pc_bound", False):
        vp = ctypes.c_void_p
        L.ocpqp_pc_create.argtypes = [ctypes.POINTER(nat.OcpQpDimC), ctypes.c_int32, ctypes.POINTER(vp)]
        L.ocpqp_pc_destroy.argtypes = [vp]
        L.ocpqp_pc_dims.argtypes = [vp, vp, vp, vp, vp, vp]
        L.ocpqp_pc_condense.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(nat.OcpQpDataC),
                                        ctypes.POINTER(nat.OcpQpDataC), vp]
        L.ocpqp_pc_expand.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(nat.OcpQpDataC),
                                      ctypes.POINTER(nat.OcpIterC), ctypes.POINTER(nat.OcpIterC), vp]
        L.ocpqp_pc_last_error.restype = ctypes.c_char_p
        for f in ("ocpqp_pc_create", "ocpqp_pc_destroy", "ocpqp_pc_dims", "ocpqp_pc_condense",
                  "ocpqp_pc_expand"):
            getattr(L, f).restype = ctypes.c_int
        L._pc_bound = True
    return L


def _check(rc):
    if rc >= 0:
        return rc
    msg = _lib().ocpqp_pc_last_error().decode(errors="replace")
    if rc == -1:
        raise InvalidBlockSize(msg)
    if rc == -3:
        raise NotImplementedError(msg)
    if rc == -5:
        raise ValueError(msg)
    raise NativeLibraryError(f"partial condensing error {rc}: {msg}")


class PartialCondensingMap:
    """Block structure of one partial condensing (reference PartialCondensingMap)."""

    def __init__(self, batch_struct, N1):
        if int(N1) < 1:
            raise InvalidBlockSize("block size must be >= 1")
        if batch_struct.dim.N < 1:
            raise InvalidBlockSize("horizon must be >= 1 for partial condensing")
        self.N1 = int(N1)
        self.dim = batch_struct.dim
        d = batch_struct.dim
        self._dimc, self._keep = nat.make_dim_c(d, batch_struct.idxb_concat(),
                                                batch_struct.idxs_concat())
        h = ctypes.c_void_p()
        _check(_lib().ocpqp_pc_create(ctypes.byref(self._dimc), self.N1, ctypes.byref(h)))
        self.handle = h
        N2 = _check(_lib().ocpqp_pc_dims(h, None, None, None, None, None))
        arrs = [np.zeros(N2 + 1, dtype=np.int32) for _ in range(4)]
        _lib().ocpqp_pc_dims(h, *(a.ctypes.data for a in arrs), None)
        nx, nu, nb, ng = arrs
        idxb = np.zeros(max(1, int(nb.sum())), dtype=np.int32)
        _lib().ocpqp_pc_dims(h, None, None, None, None, idxb.ctypes.data)
        self.new_dim = OcpQpDim(N2, nx.tolist(), nu.tolist(), nb.tolist(), ng.tolist(),
                                [0] * (N2 + 1))
        self.new_idxb = []
        o = 0
        for k in range(N2 + 1):
            self.new_idxb.append(idxb[o: o + int(nb[k])].copy())
            o += int(nb[k])
        self.starts = list(range(0, d.N, self.N1)) + [d.N]

    def close(self):
        if getattr(self, "handle", None):
            _lib().ocpqp_pc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_MAPS = {}


def _map_for(batch, N1):
    key = (batch.structure_key(), int(N1))
    m = _MAPS.get(key)
    if m is None:
        m = PartialCondensingMap(batch, N1)
        _MAPS[key] = m
    return m


def _device_full(batch, device):
    """Device batch whose every field is materialised (kernels read all fields)."""
    import torch

    out = OcpQpBatch(batch.dim, batch.B, batch.idxb, batch.idxs)
    for name in FIELD_ORDER:
        L = batch.layout.field_len[name]
        arr = batch.fields.get(name)
        if arr is None:
            t = torch.full((1, max(1, L)), default_fill(name), dtype=torch.float64, device=device)
        elif isinstance(arr, np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
        else:
            t = arr.to(device=device, dtype=torch.float64).contiguous()
        out.fields[name] = t
    return out


def _data_c_full(b):
    d = nat.OcpQpDataC()
    for i, name in enumerate(FIELD_ORDER):
        arr = b.fields[name]
        d.ptr[i] = arr.data_ptr()
        d.batch_stride[i] = 0 if arr.shape[0] == 1 else b.layout.field_len[name]
    return d


def partial_condense_batch(batch, N1, device="cuda"):
    """Condensed device batch (horizon ceil(N/N1)) and its map."""
    import torch

    from .solver import _as_batch

    batch = _as_batch(batch, check=False)
    pmap = _map_for(batch, N1)
    src = _device_full(batch, device)
    out = OcpQpBatch(pmap.new_dim, batch.B, pmap.new_idxb, None)
    lay = out.layout
    dout = nat.OcpQpDataC()
    keep = []
    for i, name in enumerate(FIELD_ORDER):
        L = lay.field_len[name]
        buf = torch.zeros((batch.B, max(1, L)), dtype=torch.float64, device=device)
        keep.append(buf)
        dout.ptr[i] = buf.data_ptr()
        dout.batch_stride[i] = max(1, L)
        if L:
            out.fields[name] = buf  # [B, L], contiguous: batch stride L
    din = _data_c_full(src)
    s = torch.cuda.current_stream(device)
    _check(_lib().ocpqp_pc_condense(pmap.handle, batch.B, ctypes.byref(din), ctypes.byref(dout),
                                    ctypes.c_void_p(s.cuda_stream)))
    del keep
    return out, pmap


def partial_expand_batch(short, pmap, batch, device="cuda"):
    """Full-horizon (y, pi, lam, t) device tensors from a condensed solution.

    ``short`` is a BatchReport of the condensed batch or a (y, pi, lam, t) tuple.
    """
    import torch

    from .solver import _as_batch

    batch = _as_batch(batch, check=False)
    src = _device_full(batch, device)
    parts = (short.y, short.pi, short.lam, short.t) if hasattr(short, "lam") else tuple(short)
    f64 = dict(dtype=torch.float64, device=device)
    sy, spi, slam, st = (torch.as_tensor(a, **f64).reshape(batch.B, -1).contiguous() for a in parts)
    lay = batch.layout
    y = torch.zeros((batch.B, lay.ny), **f64)
    pi = torch.zeros((batch.B, max(1, lay.ne)), **f64)
    lam = torch.zeros((batch.B, max(1, lay.nc)), **f64)
    t = torch.zeros((batch.B, max(1, lay.nc)), **f64)
    din = _data_c_full(src)
    s_it = nat.OcpIterC(sy.data_ptr(), spi.data_ptr(), slam.data_ptr(), st.data_ptr())
    f_it = nat.OcpIterC(y.data_ptr(), pi.data_ptr(), lam.data_ptr(), t.data_ptr())
    s = torch.cuda.current_stream(device)
    _check(_lib().ocpqp_pc_expand(pmap.handle, batch.B, ctypes.byref(din), ctypes.byref(s_it),
                                  ctypes.byref(f_it), ctypes.c_void_p(s.cuda_stream)))
    return y, pi[:, : lay.ne], lam[:, : lay.nc], t[:, : lay.nc]


def partial_condense(qp, N1):
    """Single-QP drop-in: ``(OcpQp, PartialCondensingMap)`` (condensing.py:451)."""
    if not isinstance(qp, OcpQp):
        raise TypeError("partial_condense expects an OcpQp")
    if int(N1) < 1:
        raise InvalidBlockSize("block size must be >= 1")
    if qp.dim.N < 1:
        raise InvalidBlockSize("horizon must be >= 1 for partial condensing")
    b = OcpQpBatch.from_qps([qp])
    cb, pmap = partial_condense_batch(b, N1)
    pmap._source_batch = b
    return cb.numpy().qp(0), pmap


def partial_expand(sol_p, pmap, qp):
    """Single-QP drop-in: full-horizon QpSolution (condensing.py:553)."""
    b = OcpQpBatch.from_qps([qp])
    y, pi, lam, t = partial_expand_batch(
        tuple(np.asarray(a)[None] for a in (sol_p.y, sol_p.pi, sol_p.lam, sol_p.t)), pmap, b)
    return QpSolution(b.layout, y[0].cpu().numpy(), pi[0].cpu().numpy(), lam[0].cpu().numpy(),
                      t[0].cpu().numpy())
