"""ctypes wrapper of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module; the product package never does.
See ocpqp_oracle.c for what it restates and how it is pinned to the reference.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle_ocpqp.so"

_lib = None


def build(force=False):
    src = HERE / "ocpqp_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        vp = ctypes.c_void_p
        _lib.oracle_solve.argtypes = [vp, ctypes.c_int32, vp, vp, vp, vp, ctypes.c_int32]
        _lib.oracle_residuals.argtypes = [vp, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp]
        _lib.oracle_newton_step.argtypes = [vp, ctypes.c_int32, vp, ctypes.c_double, vp, vp, vp,
                                            vp, vp, vp, vp, vp]
        for f in ("oracle_solve", "oracle_residuals", "oracle_newton_step"):
            getattr(_lib, f).restype = ctypes.c_int
    return _lib


def _structs():
    from paper_2003_02547_b200 import _native as nat

    return nat


def solve(batch, arg, nthreads=None, trace=True, guess=None):
    """Oracle solve of a host OcpQpBatch; returns a dict of numpy arrays.

    ``guess`` = (y, pi, lam, t) [B, n] arrays seeds ``arg.warm_start``
    (solver.py:113-142); without it the solve is cold."""
    nat = _structs()
    b = batch.numpy()
    lay = b.layout
    B = b.B
    nthreads = nthreads or os.cpu_count() or 1
    dimc, keep = nat.make_dim_c(b.dim, b.idxb_concat(), b.idxs_concat())
    dc = nat.data_c(b)
    from dataclasses import replace

    if guess is None and arg.warm_start != "none":
        arg = replace(arg, warm_start="none")
    carg = nat.arg_to_c(arg)
    out = dict(y=np.zeros((B, lay.ny)), pi=np.zeros((B, lay.ne)), lam=np.zeros((B, lay.nc)),
               t=np.zeros((B, lay.nc)), status=np.zeros(B, dtype=np.int32),
               iters=np.zeros(B, dtype=np.int32), res=np.zeros((B, 5)),
               flops=np.zeros(B, dtype=np.int64),
               trace=np.zeros((B, max(1, arg.iter_max), 8)) if trace else None)
    if guess is not None:
        for k, a in zip(("y", "pi", "lam", "t"), guess):
            out[k][:] = np.asarray(a, dtype=np.float64).reshape(B, -1)
    it = nat.OcpIterC(out["y"].ctypes.data, out["pi"].ctypes.data, out["lam"].ctypes.data,
                      out["t"].ctypes.data)
    st = nat.OcpStatsC(out["status"].ctypes.data, out["iters"].ctypes.data, out["res"].ctypes.data,
                       out["flops"].ctypes.data,
                       out["trace"].ctypes.data if trace else None)
    rc = lib().oracle_solve(ctypes.addressof(dimc), B, ctypes.addressof(dc), ctypes.addressof(carg),
                            ctypes.addressof(it), ctypes.addressof(st), int(nthreads))
    del keep
    if rc:
        raise RuntimeError("oracle_solve failed")
    return out


def residuals(batch, y, pi, lam, t):
    nat = _structs()
    b = batch.numpy()
    lay = b.layout
    B = b.B
    dimc, keep = nat.make_dim_c(b.dim, b.idxb_concat(), b.idxs_concat())
    dc = nat.data_c(b)
    arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(B, -1)) for a in (y, pi, lam, t)]
    pt = nat.OcpIterC(*(a.ctypes.data for a in arrs))
    out = dict(r_g=np.zeros((B, lay.ny)), r_b=np.zeros((B, lay.ne)), r_d=np.zeros((B, lay.nc)),
               r_m=np.zeros((B, lay.nc)), norms=np.zeros((B, 5)))
    rc = lib().oracle_residuals(ctypes.addressof(dimc), B, ctypes.addressof(dc), ctypes.addressof(pt),
                                out["r_g"].ctypes.data, out["r_b"].ctypes.data,
                                out["r_d"].ctypes.data, out["r_m"].ctypes.data,
                                out["norms"].ctypes.data)
    del keep
    if rc:
        raise RuntimeError("oracle_residuals failed")
    return out


def newton_step(batch, lam, t, r_g, r_b, r_d, r_m, reg=0.0, want_P=False):
    nat = _structs()
    b = batch.numpy()
    lay = b.layout
    B = b.B
    dimc, keep = nat.make_dim_c(b.dim, b.idxb_concat(), b.idxs_concat())
    dc = nat.data_c(b)
    f = [np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(B, -1))
         for a in (lam, t, r_g, r_b, r_d, r_m)]
    it = nat.OcpIterC(None, None, f[0].ctypes.data, f[1].ctypes.data)
    out = dict(dy=np.zeros((B, lay.ny)), dpi=np.zeros((B, lay.ne)), dlam=np.zeros((B, lay.nc)),
               dt=np.zeros((B, lay.nc)), fail=np.zeros(B, dtype=np.int32))
    stp = nat.OcpIterC(out["dy"].ctypes.data, out["dpi"].ctypes.data, out["dlam"].ctypes.data,
                       out["dt"].ctypes.data)
    Pn = int(sum(int(x) ** 2 for x in b.dim.nx))
    P = np.zeros((B, Pn)) if want_P else None
    rc = lib().oracle_newton_step(ctypes.addressof(dimc), B, ctypes.addressof(dc), float(reg),
                                  ctypes.addressof(it), f[2].ctypes.data, f[3].ctypes.data,
                                  f[4].ctypes.data, f[5].ctypes.data, ctypes.addressof(stp),
                                  out["fail"].ctypes.data, P.ctypes.data if want_P else None)
    del keep
    if rc:
        raise RuntimeError("oracle_newton_step failed")
    if want_P:
        out["P"] = P
    return out
