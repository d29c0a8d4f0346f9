"""The C-ABI library loads and exports everything include/ocpqp_b200.h declares.

Runs without a GPU: only symbol presence, the pure-host layout entry point and
clean error returns are exercised here (no compute calls).
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2003_02547_b200 import OcpLayout, OcpQpDim
from paper_2003_02547_b200 import _native as nat
from paper_2003_02547_b200 import build as pkg_build
from paper_2003_02547_b200.layout import FIELD_ORDER

HEADER = Path(__file__).resolve().parents[1] / "include" / "ocpqp_b200.h"


@pytest.fixture(scope="module")
def lib():
    pkg_build.build()
    return nat.lib()


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ocpqp_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for n in ("ocpqp_plan_create", "ocpqp_solve", "ocpqp_solve_host", "ocpqp_newton_step",
              "ocpqp_residuals", "ocpqp_layout", "ocpqp_last_error"):
        assert n in names
    assert set(names) == set(nat.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.ocpqp_abi_version() == 2


def test_enum_order_matches_host_field_order():
    text = HEADER.read_text()
    body = text[text.index("enum OcpQpField"):text.index("OCPQP_NUM_FIELDS")]
    names = re.findall(r"OCPQP_F_(\w+)", body)
    assert tuple(names) == FIELD_ORDER


def test_layout_entry_matches_python_layout(lib):
    d = OcpQpDim(3, nx=[4, 4, 3, 3], nu=[2, 1, 1, 0], nb=[3, 5, 2, 3], ng=[1, 0, 2, 1],
                 ns=[1, 0, 1, 0])
    idxb = np.concatenate([np.arange(3), np.arange(5), np.arange(2), np.arange(3)])
    idxs = np.array([0, 1])
    dimc, keep = nat.make_dim_c(d, idxb, idxs)
    out = (ctypes.c_int64 * (6 + len(FIELD_ORDER)))()
    assert lib.ocpqp_layout(ctypes.byref(dimc), out, len(out)) == 0
    L = OcpLayout(d)
    assert (out[0], out[1], out[2], out[3], out[4]) == (L.ny, L.ne, L.nc, L.nv, L.ns_tot)
    for i, name in enumerate(FIELD_ORDER):
        assert out[6 + i] == L.field_len[name], name


def test_layout_entry_rejects_bad_structure(lib):
    d = OcpQpDim(1, nx=[2, 2], nu=[1, 0], nb=[3, 2])
    dimc, keep = nat.make_dim_c(d, np.array([2, 1, 0, 0, 1]), np.zeros(0))
    out = (ctypes.c_int64 * 40)()
    rc = lib.ocpqp_layout(ctypes.byref(dimc), out, 40)
    assert rc == -2  # DimensionMismatch: idxb not strictly increasing
    assert b"strictly increasing" in lib.ocpqp_last_error()
    with pytest.raises(Exception):
        nat.check(rc)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2003_02547_b200 as pkg
    from paper_2003_02547_b200.generators import make_batch

    with pytest.raises(pkg.NativeLibraryError):
        pkg.solve_ocp_qp_batch(make_batch(0), pkg.mode_preset("speed"))


def test_dense_plan_rejects_bad_structure_without_gpu_work(lib):
    """ocpqp_dense_plan_create validates before touching the device."""
    dim = nat.OcpDenseDimC(4, 5, 0, 0, 0, None)       # ne > nv
    h = ctypes.c_void_p()
    assert lib.ocpqp_dense_plan_create(ctypes.byref(dim), 1, 0, ctypes.byref(h)) == -1
    ib = (ctypes.c_int32 * 2)(1, 0)
    dim = nat.OcpDenseDimC(4, 1, 2, 0, 0, ib)           # idxb not increasing
    assert lib.ocpqp_dense_plan_create(ctypes.byref(dim), 1, 0, ctypes.byref(h)) == -2
    dim = nat.OcpDenseDimC(4, 1, 0, 0, 1, None)         # soft rows
    assert lib.ocpqp_dense_plan_create(ctypes.byref(dim), 1, 0, ctypes.byref(h)) == -3
    assert b"soft rows" in lib.ocpqp_last_error()


def test_dense_eq_residual_assembly_at_reference_solution(golden):
    """Host-side report assembly (dense.py _dense_residuals, view.py:272-288 on
    the DenseView) reproduces the reference's final residual norms at the
    reference's own solutions."""
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_gpu_dense_eq import build, cases

    from paper_2003_02547_b200.dense import _dense_residuals

    g = golden("dense_eq")
    for seed, nv, ne, nb, ng, method, rd in cases():
        p = f"e{seed}"
        if int(g[f"{p}_status"]) != 0:
            continue
        q = build(seed, nv, ne, nb, ng, rd)
        r = _dense_residuals(q, g[f"{p}_y"], g[f"{p}_pi"], g[f"{p}_lam"], g[f"{p}_t"])
        got = np.array([r.res_g, r.res_b, r.res_d, r.res_m, r.mu])
        ref = g[f"{p}_res"]
        assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref))), (seed, got, ref)
