"""Batched partial / full condensing and expansion on the GPU (reference
condensing.py:160-619).

``partial_condense_batch(batch, N1)`` turns a batch of OCP-QPs with horizon N
into the batch of block-condensed QPs with horizon ceil(N / N1) (each block of
N1 stages condensed with its initial state kept; the old terminal stage carried
over verbatim), and ``partial_expand_batch`` maps the short-horizon solutions
back to the full horizon (forward state rollout, multiplier routing, costate
recursion for pi).  The routing tables are built once per structure by the C
ABI (ocpqp_pc_create); the arithmetic runs in the CUDA kernels of
csrc/ocpqp_condense.cu.  ``partial_condense`` / ``partial_expand`` are the
reference's single-QP calls.

``condense_batch(batch, keep_x0)`` is full condensing (condense,
condensing.py:160-340): every state except (optionally) x0 eliminated, the
dense QP returned as the single-stage batch (N = 0, nx = 0, nu = nv) that the
IPM kernels solve exactly like the reference's dense backend (dense.py);
``expand_batch`` is expand_solution (condensing.py:343-429).  ``condense`` /
``expand_solution`` are the single-QP drop-ins.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .batch import OcpQpBatch, default_fill
from .errors import (CondenseError, DimensionMismatch, InvalidBlockSize, NativeLibraryError,
                     NotPositiveDefinite, RankDeficient)
from .layout import FIELD_ORDER, QpSolution
from .qp_data import OcpQp, OcpQpDim

__all__ = ["PartialCondensingMap", "partial_condense_batch", "partial_expand_batch",
           "partial_condense", "partial_expand", "CondensingMap", "condense_batch", "expand_batch",
           "condense", "expand_solution", "detect_fixed_x0"]


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
        L.ocpqp_fc_create.argtypes = [ctypes.POINTER(nat.OcpQpDimC), ctypes.c_int32, ctypes.c_int32,
                                      vp, vp, ctypes.POINTER(vp)]
        L.ocpqp_fc_create.restype = ctypes.c_int
        L.ocpqp_pc_soft.argtypes = [vp, vp, vp]
        L.ocpqp_pc_set_variant.argtypes = [vp, ctypes.c_int32]
        L.ocpqp_pc_soft.restype = ctypes.c_int
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
    if rc == -6:
        raise CondenseError(msg)
    if rc == -7:
        raise NotPositiveDefinite(msg)
    if rc == -8:
        raise RankDeficient(msg)
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
        ns, self.new_idxs = _soft_of(h, N2)
        self.new_dim = OcpQpDim(N2, nx.tolist(), nu.tolist(), nb.tolist(), ng.tolist(), ns.tolist())
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


def _soft_of(h, N2):
    """(ns per new stage, list of new idxs arrays) of a condensing plan."""
    ns = np.zeros(N2 + 1, dtype=np.int32)
    tot = _check(_lib().ocpqp_pc_soft(h, ns.ctypes.data, None))
    flat = np.zeros(max(1, tot), dtype=np.int32)
    _lib().ocpqp_pc_soft(h, None, flat.ctypes.data)
    out, o = [], 0
    for k in range(N2 + 1):
        out.append(flat[o: o + int(ns[k])].copy())
        o += int(ns[k])
    return ns, out


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
    out = OcpQpBatch(pmap.new_dim, batch.B, pmap.new_idxb, pmap.new_idxs)
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


# ---------------------------------------------------------------------------
# full condensing (condensing.py:160-429)
# ---------------------------------------------------------------------------

def _stage0_rows(batch):
    """Host copies [Bf, nb0] of the stage-0 lb, ub, maskl, masku of a batch
    (one device-to-host copy for a device batch)."""
    from .batch import default_fill

    d = batch.dim
    nb0 = int(d.nb[0])
    names = ("lb", "ub", "maskl", "masku")
    parts, dev = [], None
    for name in names:
        arr = batch.fields.get(name)
        if arr is None:
            parts.append(None)
            continue
        a = arr[:, batch.layout.stage_slice(name, 0)][:, :nb0]
        if not isinstance(a, np.ndarray):
            dev = a
        parts.append(a)
    if dev is not None:
        import torch

        rows = max(p.shape[0] for p in parts if p is not None)
        stk = torch.stack([torch.as_tensor(p, dtype=torch.float64, device=dev.device).expand(rows, nb0)
                           if p is not None else
                           torch.full((rows, nb0), default_fill(n), dtype=torch.float64,
                                      device=dev.device)
                           for p, n in zip(parts, names)])
        host = stk.cpu().numpy()
        return [host[i] for i in range(len(names))]
    return [np.asarray(p, dtype=np.float64) if p is not None else np.full((1, nb0), default_fill(n))
            for p, n in zip(parts, names)]


def detect_fixed_x0(batch):
    """(all_fixed, fix_rows) of _detect_fixed_x0 (condensing.py:97-118) for a batch.

    A stage-0 x row fixes its component when lb == ub, finite, both masks set.
    Every QP of the batch must fix the same rows (CondenseError otherwise).
    """
    d = batch.dim
    nu0, nx0 = int(d.nu[0]), int(d.nx[0])
    lb, ub, ml, mu = _stage0_rows(batch)
    fixed = (lb == ub) & np.isfinite(lb) & (ml != 0.0) & (mu != 0.0)
    B = batch.B
    fixed = np.broadcast_to(fixed, (B, fixed.shape[1])) if fixed.shape[0] == 1 else fixed
    idxb = batch.idxb[0]
    xrow = idxb >= nu0
    fixed = fixed & xrow[None, :]
    if B > 1 and not np.all(fixed == fixed[:1]):
        raise CondenseError("the QPs of the batch fix different initial-state rows; "
                            "condense them separately")
    rows = [(int(i), int(idxb[i]) - nu0) for i in np.flatnonzero(fixed[0])]
    comps = {c for _, c in rows}
    all_fixed = (len(comps) == nx0) if nx0 else True
    return all_fixed, rows


class CondensingMap:
    """Full-condensing plan of one batch structure (reference CondensingMap)."""

    def __init__(self, batch, keep_x0=None):
        d = batch.dim
        all_fixed, rows = detect_fixed_x0(batch)
        if keep_x0 is None:
            keep_x0 = not all_fixed
        if not keep_x0 and not all_fixed:
            raise CondenseError("keep_x0=False requires every initial-state component fixed "
                                "by active equal-bound box rows")
        self.keep_x0 = bool(keep_x0)
        self.fix_rows = [] if self.keep_x0 else rows
        self.dim = d
        self.N = d.N
        self.nx0 = int(d.nx[0])
        self._dimc, self._keep = nat.make_dim_c(d, batch.idxb_concat(), batch.idxs_concat())
        fr = np.array([r for r, _ in self.fix_rows] or [0], dtype=np.int32)
        fc = np.array([c for _, c in self.fix_rows] or [0], dtype=np.int32)
        h = ctypes.c_void_p()
        _check(_lib().ocpqp_fc_create(ctypes.byref(self._dimc), int(self.keep_x0),
                                      len(self.fix_rows), fr.ctypes.data, fc.ctypes.data,
                                      ctypes.byref(h)))
        self.handle = h
        arrs = [np.zeros(1, dtype=np.int32) for _ in range(4)]
        _lib().ocpqp_pc_dims(h, *(a.ctypes.data for a in arrs), None)
        nx, nu, nb, ng = (int(a[0]) for a in arrs)
        idxb = np.zeros(max(1, nb), dtype=np.int32)
        _lib().ocpqp_pc_dims(h, None, None, None, None, idxb.ctypes.data)
        self.nv = nu
        ns, self.new_idxs = _soft_of(h, 0)
        self.new_dim = OcpQpDim(0, [0], [nu], [nb], [ng], [int(ns[0])])
        self.new_idxb = [idxb[:nb].copy()]
        zx = self.nx0 if self.keep_x0 else 0
        self.u_off, off = [], zx
        for n in range(d.N + 1):
            self.u_off.append(off if int(d.nu[n]) else None)
            off += int(d.nu[n])

    def close(self):
        if getattr(self, "handle", None):
            _lib().ocpqp_pc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_FMAPS = {}


def _fmap_for(batch, keep_x0):
    all_fixed, rows = detect_fixed_x0(batch)
    keep = (not all_fixed) if keep_x0 is None else bool(keep_x0)
    key = (batch.structure_key(), keep, tuple(rows) if not keep else ())
    m = _FMAPS.get(key)
    if m is None:
        m = CondensingMap(batch, keep)
        _FMAPS[key] = m
    return m


def condense_batch(batch, keep_x0=None, device="cuda", variant="classical"):
    """Fully condensed device batch (N = 0, nx = 0, nu = nv) and its map.

    ``variant``: the cost recursion of the reference's ``condense``
    (condensing.py:128-157): "classical" (explicit P) or "square_root"
    (Cholesky / QR factors of P; raises NotPositiveDefinite / RankDeficient
    like the reference when a stage cost Q is not positive definite)."""
    import torch

    from .solver import _as_batch

    if variant not in ("classical", "square_root"):
        raise ValueError(f"unknown condensing variant '{variant}'")
    batch = _as_batch(batch, check=False)
    cmap = _fmap_for(batch, keep_x0)
    _check(_lib().ocpqp_pc_set_variant(cmap.handle, 1 if variant == "square_root" else 0))
    src = _device_full(batch, device)
    out = OcpQpBatch(cmap.new_dim, batch.B, cmap.new_idxb, cmap.new_idxs)
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
            out.fields[name] = buf
    din = _data_c_full(src)
    s = torch.cuda.current_stream(device)
    _check(_lib().ocpqp_pc_condense(cmap.handle, batch.B, ctypes.byref(din), ctypes.byref(dout),
                                    ctypes.c_void_p(s.cuda_stream)))
    del keep
    return out, cmap


def expand_batch(dense, cmap, batch, device="cuda"):
    """Full OCP (y, pi, lam, t) device tensors from dense solutions
    (expand_solution, condensing.py:343-429).  ``dense`` is a BatchReport of
    the condensed batch or a (y, pi, lam, t) tuple."""
    import torch

    from .solver import _as_batch

    batch = _as_batch(batch, check=False)
    src = _device_full(batch, device)
    parts = (dense.y, dense.pi, dense.lam, dense.t) if hasattr(dense, "lam") else tuple(dense)
    f64 = dict(dtype=torch.float64, device=device)

    def dev(a):
        a = torch.as_tensor(a, **f64)
        if a.numel() == 0:  # pi of the N = 0 form is empty
            return torch.zeros((batch.B, 1), **f64)
        return a.reshape(batch.B, -1).contiguous()

    sy, spi, slam, st = (dev(a) for a in parts)
    if sy.shape[1] < cmap.nv:
        raise DimensionMismatch("dense solution does not match the map")
    lay = batch.layout
    y = torch.zeros((batch.B, lay.ny), **f64)
    pi = torch.zeros((batch.B, max(1, lay.ne)), **f64)
    lam = torch.zeros((batch.B, max(1, lay.nc)), **f64)
    t = torch.zeros((batch.B, max(1, lay.nc)), **f64)
    din = _data_c_full(src)
    s_it = nat.OcpIterC(sy.data_ptr(), spi.data_ptr(), slam.data_ptr(), st.data_ptr())
    f_it = nat.OcpIterC(y.data_ptr(), pi.data_ptr(), lam.data_ptr(), t.data_ptr())
    s = torch.cuda.current_stream(device)
    _check(_lib().ocpqp_pc_expand(cmap.handle, batch.B, ctypes.byref(din), ctypes.byref(s_it),
                                  ctypes.byref(f_it), ctypes.c_void_p(s.cuda_stream)))
    return y, pi[:, : lay.ne], lam[:, : lay.nc], t[:, : lay.nc]


def condense(qp, keep_x0=None, variant="classical"):
    """Single-QP drop-in: ``(DenseQp, CondensingMap)`` (condensing.py:160)."""
    from .dense import ocp_to_dense

    if not isinstance(qp, OcpQp):
        raise TypeError("condense expects an OcpQp")
    b = OcpQpBatch.from_qps([qp])
    cb, cmap = condense_batch(b, keep_x0, variant=variant)
    return ocp_to_dense(cb.numpy().qp(0)), cmap


def expand_solution(dense_sol, cmap, qp, pi_terminal=None):
    """Single-QP drop-in: full OCP QpSolution (condensing.py:343)."""
    if pi_terminal is not None:
        raise NotImplementedError("pi_terminal seeding is used by partial condensing only")
    if dense_sol.v.shape[0] != cmap.nv:
        raise DimensionMismatch("dense solution does not match the map")
    b = OcpQpBatch.from_qps([qp])
    y, pi, lam, t = expand_batch(
        tuple(np.asarray(a)[None] for a in (dense_sol.y, dense_sol.pi, dense_sol.lam, dense_sol.t)),
        cmap, b)
    return QpSolution(b.layout, y[0].cpu().numpy(), pi[0].cpu().numpy(), lam[0].cpu().numpy(),
                      t[0].cpu().numpy())
