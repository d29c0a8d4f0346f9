"""ctypes binding of the CUDA library's C ABI (include/ocpqp_b200.h).

The library is built in-tree (``paper_2003_02547_b200/_lib/libocpqp_b200.so``,
see build.py).  There is no CPU fallback: if the library is missing or fails
to load, every solve raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import (
    DimensionMismatch,
    InvalidDim,
    NativeLibraryError,
)
from .layout import FIELD_ORDER

__all__ = ["lib", "LIB_PATH", "OcpQpDimC", "OcpQpDataC", "OcpIpmArgC", "OcpIterC",
           "OcpStatsC", "Plan", "EXPORTED_SYMBOLS", "make_dim_c", "arg_to_c", "check"]

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libocpqp_b200.so"
NF = len(FIELD_ORDER)

EXPORTED_SYMBOLS = (
    "ocpqp_layout", "ocpqp_plan_create", "ocpqp_plan_destroy", "ocpqp_solve",
    "ocpqp_solve_host", "ocpqp_residuals", "ocpqp_newton_step", "ocpqp_factor_export",
    "ocpqp_plan_info", "ocpqp_fp64_peak", "ocpqp_abi_version", "ocpqp_last_error",
    "ocpqp_pc_create", "ocpqp_pc_destroy", "ocpqp_pc_dims", "ocpqp_pc_condense",
    "ocpqp_pc_expand", "ocpqp_pc_last_error", "ocpqp_shift_guess", "ocpqp_fc_create",
    "ocpqp_pc_soft", "ocpqp_pc_set_variant", "ocpqp_plan_dispatch_hint", "ocpqp_dense_plan_create", "ocpqp_dense_plan_destroy", "ocpqp_dense_solve",
)

_i32p = ctypes.POINTER(ctypes.c_int32)


class OcpQpDimC(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("nx", _i32p), ("nu", _i32p), ("nb", _i32p),
                ("ng", _i32p), ("ns", _i32p), ("idxb", _i32p), ("idxs", _i32p)]


class OcpQpDataC(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p * NF), ("batch_stride", ctypes.c_int64 * NF)]


class OcpIpmArgC(ctypes.Structure):
    _fields_ = [("iter_max", ctypes.c_int32), ("pred_corr", ctypes.c_int32),
                ("cond_pred_corr", ctypes.c_int32), ("warm_start", ctypes.c_int32),
                ("alpha_min", ctypes.c_double), ("mu0", ctypes.c_double),
                ("tol_stat", ctypes.c_double), ("tol_eq", ctypes.c_double),
                ("tol_ineq", ctypes.c_double), ("tol_comp", ctypes.c_double),
                ("reg_prim", ctypes.c_double), ("lam_min", ctypes.c_double),
                ("t_min", ctypes.c_double), ("t0", ctypes.c_double),
                ("corr_ratio", ctypes.c_double), ("ftb", ctypes.c_double),
                # ABI v2: modes beyond speed
                ("itref_pred_max", ctypes.c_int32), ("itref_corr_max", ctypes.c_int32),
                ("use_qr_fallback", ctypes.c_int32), ("use_qr_always", ctypes.c_int32),
                ("riccati_variant", ctypes.c_int32), ("abs_form", ctypes.c_int32),
                ("comp_res_pred", ctypes.c_int32), ("mu_only_exit", ctypes.c_int32),
                ("itref_stop_ratio", ctypes.c_double), ("qr_fallback_ratio", ctypes.c_double)]


class OcpDenseDimC(ctypes.Structure):
    _fields_ = [("nv", ctypes.c_int32), ("ne", ctypes.c_int32), ("nb", ctypes.c_int32),
                ("ng", ctypes.c_int32), ("ns", ctypes.c_int32), ("idxb", _i32p)]


DENSE_FIELDS = ("H", "g", "A", "b", "lb", "ub", "C", "lg", "ug", "maskl", "masku")


class OcpDenseDataC(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in DENSE_FIELDS] + [
        ("batch_stride", ctypes.c_int64 * len(DENSE_FIELDS))]


class OcpIterC(ctypes.Structure):
    _fields_ = [("y", ctypes.c_void_p), ("pi", ctypes.c_void_p), ("lam", ctypes.c_void_p),
                ("t", ctypes.c_void_p)]


class OcpStatsC(ctypes.Structure):
    _fields_ = [("status", ctypes.c_void_p), ("iterations", ctypes.c_void_p),
                ("res", ctypes.c_void_p), ("flops", ctypes.c_void_p),
                ("trace", ctypes.c_void_p)]


_LIB = None


def lib():
    """Load the CUDA library once; raise loudly if it is not there."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("OCPQP_B200_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryError(
            f"CUDA library {path} is missing; run `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (no CPU fallback exists)")
    try:
        L = ctypes.CDLL(str(path))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    vp = ctypes.c_void_p
    L.ocpqp_layout.argtypes = [ctypes.POINTER(OcpQpDimC), ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]
    L.ocpqp_plan_create.argtypes = [ctypes.POINTER(OcpQpDimC), ctypes.c_int32, ctypes.POINTER(vp)]
    L.ocpqp_plan_destroy.argtypes = [vp]
    L.ocpqp_plan_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]
    L.ocpqp_solve.argtypes = [vp, ctypes.POINTER(OcpQpDataC), ctypes.POINTER(OcpIpmArgC),
                              ctypes.POINTER(OcpIterC), ctypes.POINTER(OcpStatsC), vp]
    L.ocpqp_solve_host.argtypes = L.ocpqp_solve.argtypes
    L.ocpqp_residuals.argtypes = [vp, ctypes.POINTER(OcpQpDataC), ctypes.POINTER(OcpIterC),
                                  vp, vp, vp, vp, vp, vp]
    L.ocpqp_newton_step.argtypes = [vp, ctypes.POINTER(OcpQpDataC), ctypes.c_double,
                                    ctypes.POINTER(OcpIterC), vp, vp, vp, vp,
                                    ctypes.POINTER(OcpIterC), vp, vp]
    L.ocpqp_factor_export.argtypes = [vp, ctypes.c_int32, vp, vp]
    L.ocpqp_shift_guess.argtypes = [vp, ctypes.POINTER(OcpQpDataC), ctypes.POINTER(OcpIterC),
                                    ctypes.POINTER(OcpIterC), vp]
    L.ocpqp_dense_plan_create.argtypes = [ctypes.POINTER(OcpDenseDimC), ctypes.c_int32,
                                          ctypes.c_int32, ctypes.POINTER(vp)]
    L.ocpqp_dense_plan_destroy.argtypes = [vp]
    L.ocpqp_dense_solve.argtypes = [vp, ctypes.POINTER(OcpDenseDataC), ctypes.POINTER(OcpIpmArgC),
                                    ctypes.c_double, ctypes.POINTER(OcpIterC),
                                    ctypes.POINTER(OcpStatsC), vp]
    L.ocpqp_abi_version.argtypes = []
    L.ocpqp_last_error.argtypes = []
    L.ocpqp_last_error.restype = ctypes.c_char_p
    for name in EXPORTED_SYMBOLS:
        if name not in ("ocpqp_last_error", "ocpqp_pc_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _LIB = L
    return L


def check(rc):
    """Map a C ABI return code to the reference's exception classes."""
    if rc == 0:
        return
    msg = lib().ocpqp_last_error().decode(errors="replace")
    if rc == -1:
        raise InvalidDim(msg)
    if rc == -2:
        raise DimensionMismatch(msg)
    if rc == -3:
        raise NotImplementedError(msg)
    if rc == -5:
        raise ValueError(msg)
    raise NativeLibraryError(f"ocpqp error {rc}: {msg}")


def make_dim_c(dim, idxb_concat, idxs_concat):
    """OcpQpDimC plus the numpy arrays that must stay alive with it."""
    keep = [np.ascontiguousarray(np.asarray(a, dtype=np.int32))
            for a in (dim.nx, dim.nu, dim.nb, dim.ng, dim.ns, idxb_concat, idxs_concat)]
    # non-empty buffers so pointers are valid even for zero-length sets
    keep = [a if a.size else np.zeros(1, dtype=np.int32) for a in keep]
    ptrs = [a.ctypes.data_as(_i32p) for a in keep]
    c = OcpQpDimC(int(dim.N), *ptrs)
    return c, keep


def arg_to_c(arg):
    warm = {"none": 0, "primal": 1, "primal_dual": 2}[arg.warm_start]
    return OcpIpmArgC(int(arg.iter_max), int(bool(arg.pred_corr)), int(bool(arg.cond_pred_corr)),
                      warm, float(arg.alpha_min), float(arg.mu0), float(arg.tol_stat),
                      float(arg.tol_eq), float(arg.tol_ineq), float(arg.tol_comp),
                      float(arg.reg_prim), float(arg.lam_min), float(arg.t_min), float(arg.t0),
                      float(arg.corr_ratio), float(arg.ftb),
                      int(arg.itref_pred_max), int(arg.itref_corr_max),
                      int(bool(arg.use_qr_fallback)), int(bool(arg.use_qr_always)),
                      {"classical": 0, "square_root": 1}[arg.riccati_variant],
                      int(bool(arg.abs_form)), int(bool(arg.comp_res_pred)),
                      int(arg.mode == "speed_abs"),
                      float(arg.itref_stop_ratio), float(arg.qr_fallback_ratio))


def ptr_of(x):
    """Device or host address of a torch tensor / numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def data_c(batch):
    """OcpQpDataC of a packed batch (fields: torch tensors or numpy arrays).

    Cached on the batch while its field objects are unchanged."""
    sig = tuple((name, id(arr), ptr_of(arr)) for name, arr in batch.fields.items())
    cached = getattr(batch, "_datac", None)
    if cached is not None and cached[0] == sig:
        return cached[1]
    d = _data_c(batch)
    batch._datac = (sig, d)
    return d


def _data_c(batch):
    d = OcpQpDataC()
    lay = batch.layout
    for i, name in enumerate(FIELD_ORDER):
        arr = batch.fields.get(name)
        if arr is None or lay.field_len[name] == 0:
            d.ptr[i] = None
            d.batch_stride[i] = 0
            continue
        d.ptr[i] = ptr_of(arr)
        d.batch_stride[i] = 0 if arr.shape[0] == 1 else lay.field_len[name]
    return d


class Plan:
    """Owns an ``OcpPlan*`` for one (structure, batch size)."""

    def __init__(self, batch_struct, B):
        L = lib()
        self.B = int(B)
        self._dimc, self._keep = make_dim_c(batch_struct.dim, batch_struct.idxb_concat(),
                                            batch_struct.idxs_concat())
        h = ctypes.c_void_p()
        check(L.ocpqp_plan_create(ctypes.byref(self._dimc), self.B, ctypes.byref(h)))
        self.handle = h

    def info(self):
        out = (ctypes.c_int64 * 9)()
        check(lib().ocpqp_plan_info(self.handle, out, 9))
        kind = {0: "generic", 1: "team", 2: "row"}[int(out[5])]
        return dict(kernel=kind, threads_per_cta=out[0], slots=out[1], smem_bytes=out[2],
                    smem_mask=out[3], ws_doubles_per_slot=out[4], lanes_per_qp=out[6],
                    grid=out[7], store_in_smem=bool(out[8]))

    def dispatch_hint(self, on=True):
        """Hand out the next solves' QPs by this plan's previous iteration counts
        (ocpqp_plan_dispatch_hint; team kernel, repeated solves of similar batches)."""
        L = lib()
        L.ocpqp_plan_dispatch_hint.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        check(L.ocpqp_plan_dispatch_hint(self.handle, 1 if on else 0))

    def close(self):
        if getattr(self, "handle", None):
            lib().ocpqp_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
