"""Host-side API: containers, presets, layout, packing, generators (no GPU).

Mirrors the reference's own unit tests of the data model
(tests/test_qp_data.py, test_ipm_core.py presets) on this package's objects.
"""

import numpy as np
import pytest

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import (
    DimensionMismatch,
    IndexOutOfRange,
    InvalidDim,
    OcpLayout,
    OcpQp,
    OcpQpBatch,
    OcpQpDim,
    QpSolution,
    UnknownField,
    mode_preset,
    validate,
)
from paper_2003_02547_b200 import roofline as rf
from paper_2003_02547_b200.generators import CONFIGS, chain_dynamics, config_dim, make_batch
from paper_2003_02547_b200.ipm import supported_reason
from paper_2003_02547_b200.sharding import shard_range

from conftest import random_case_qp, random_cases


def small_dim():
    return OcpQpDim(2, nx=[2, 2, 2], nu=[1, 1, 0], nb=[3, 2, 1], ng=[1, 0, 1], ns=[1, 0, 0])


def test_dim_validation():
    with pytest.raises(InvalidDim):
        OcpQpDim(-1, nx=[], nu=[])
    with pytest.raises(InvalidDim):
        OcpQpDim(1, nx=[2, 2], nu=[1, 0], nb=[4, 0])      # nb > nu + nx
    with pytest.raises(InvalidDim):
        OcpQpDim(1, nx=[2, 2], nu=[1, 0], nb=[1, 0], ng=[0, 0], ns=[2, 0])
    with pytest.raises(InvalidDim):
        OcpQpDim(1, nx=[2], nu=[1, 0])                    # wrong length
    with pytest.raises(InvalidDim):
        OcpQp("not a dim")


def test_zero_init_and_roundtrip():
    qp = OcpQp(small_dim())
    assert np.all(np.isinf(qp.get_field("lb", 0))) and np.all(qp.get_field("lb", 0) < 0)
    assert np.all(qp.get_field("ub", 0) == np.inf)
    assert np.array_equal(qp.get_field("idxb", 0), np.arange(3))
    assert np.array_equal(qp.get_field("maskl", 0), np.ones(4))
    rng = np.random.default_rng(0)
    for name, n in (("Q", 0), ("S", 1), ("R", 0), ("q", 2), ("C", 0), ("D", 0), ("A", 1),
                    ("B", 0), ("b", 1), ("Zl", 0), ("lg", 2)):
        shape = qp.get_field(name, n).shape
        v = rng.standard_normal(shape)
        qp.set_field(name, n, v)
        out = qp.get_field(name, n)
        assert np.array_equal(out, v)
        out[...] = 0.0  # a copy: storage unchanged
        assert np.array_equal(qp.get_field(name, n), v)


def test_field_errors():
    qp = OcpQp(small_dim())
    with pytest.raises(UnknownField):
        qp.set_field("nope", 0, [1.0])
    with pytest.raises(IndexOutOfRange):
        qp.set_field("Q", 3, np.eye(2))
    with pytest.raises(IndexOutOfRange):
        qp.set_field("A", 2, np.eye(2))                    # dynamics only 0..N-1
    with pytest.raises(DimensionMismatch):
        qp.set_field("Q", 0, np.eye(3))


def test_virtual_box_fields():
    qp = OcpQp(OcpQpDim(1, nx=[2, 2], nu=[1, 0], nb=[3, 0]))
    qp.set_field("idxb", 0, [0, 1, 2])
    qp.set_field("lbu", 0, [-1.0])
    qp.set_field("lbx", 0, [-2.0, -3.0])
    qp.set_field("ubx", 0, [2.0, 3.0])
    assert np.array_equal(qp.get_field("lb", 0), [-1.0, -2.0, -3.0])
    assert np.array_equal(qp.get_field("lbx", 0), [-2.0, -3.0])
    assert np.array_equal(qp.get_field("ubu", 0), [np.inf])
    with pytest.raises(DimensionMismatch):
        qp.set_field("lbx", 0, [1.0])


def test_validate_rules():
    qp = OcpQp(small_dim())
    assert validate(qp) == []
    qp.set_field("Q", 0, [[1.0, 2.0], [0.0, 1.0]])
    qp.set_field("idxb", 0, [2, 1, 0])
    qp.set_field("maskl", 0, [0.5, 1, 1, 1])
    qp.set_field("Zl", 0, [-1.0])
    kinds = {v.field for v in validate(qp) if v.severity == "error"}
    assert {"Q", "idxb", "maskl", "Zl"} <= kinds
    qp2 = OcpQp(small_dim())
    qp2.set_field("lb", 1, [1.0, 1.0])
    qp2.set_field("ub", 1, [0.0, 2.0])
    assert [v.severity for v in validate(qp2)] == ["warning"]


def test_presets_and_support():
    s = mode_preset("speed")
    assert (s.abs_form, s.comp_res_pred, s.itref_corr_max, s.lam_min) == (False, True, 0, 1e-16)
    assert mode_preset("balance").use_qr_fallback and mode_preset("robust").use_qr_always
    assert mode_preset("speed_abs").abs_form
    with pytest.raises(ValueError):
        mode_preset("fast")
    t = s.with_tol(1e-6)
    assert (t.tol_stat, t.tol_eq, t.tol_ineq, t.tol_comp) == (1e-6,) * 4
    assert supported_reason(s) is None
    for m in ("speed_abs", "balance", "robust"):
        assert supported_reason(mode_preset(m)) is None
    from dataclasses import replace

    # the reference's own loop cannot run this combination (solver.py:191-216)
    bad = replace(s, comp_res_pred=False)
    assert supported_reason(bad) is not None
    with pytest.raises(NotImplementedError):
        pkg.solve_ocp_qp(OcpQp(small_dim()), bad)
    with pytest.raises(ValueError):
        pkg.IpmArg(tol_stat=0.0).validate()


def test_layout_offsets_match_reference_convention():
    L = OcpLayout(small_dim())
    # v = (u0, x0, u1, x1, x2); slots per stage 2 m + 2 ns
    assert L.u_off == [0, 3, 6] and L.x_off == [1, 4, 6]
    assert L.nv == 8 and L.ns_tot == 1 and L.ny == 10
    assert L.ne == 4 and L.pi_off == [0, 2]
    assert L.c_off == [0, 10, 14] and L.nc == 18
    sol = QpSolution(L)
    sol.y[:] = np.arange(L.ny)
    assert np.array_equal(sol.u(1), [3.0]) and np.array_equal(sol.x(2), [6.0, 7.0])
    assert np.array_equal(sol.sl(0), [8.0]) and np.array_equal(sol.su(0), [9.0])
    assert QpSolution.from_flat(L, sol.flat()).y.tolist() == sol.y.tolist()


@pytest.mark.parametrize("case", random_cases()[:3], ids=lambda c: f"seed{c[0]}")
def test_pack_unpack_roundtrip(case):
    qp = random_case_qp(*case)
    b = OcpQpBatch.from_qps([qp, qp])
    assert all(a.shape[0] == 1 for a in b.fields.values())  # identical -> broadcast
    q2 = b.qp(1)
    for n in range(qp.dim.N + 1):
        for name in ("Q", "S", "R", "q", "r", "lb", "ub", "C", "D", "lg", "ug", "idxb", "idxs",
                     "Zl", "Zu", "zl", "zu", "maskl", "masku"):
            assert np.array_equal(q2.get_field(name, n), qp.get_field(name, n)), (name, n)
    for n in range(qp.dim.N):
        for name in ("A", "B", "b"):
            assert np.array_equal(q2.get_field(name, n), qp.get_field(name, n))


def test_batch_rejects_mixed_structure():
    qa = random_case_qp(*random_cases()[0])
    qb = random_case_qp(*random_cases()[1])
    with pytest.raises(DimensionMismatch):
        OcpQpBatch.from_qps([qa, qb])


def test_generators_match_baseline_shapes():
    for cfg, spec in CONFIGS.items():
        d = config_dim(spec)
        assert d.N == spec.N and int(d.nx[0]) == spec.nx and int(d.nu[0]) == spec.nu
        assert int(d.nu[d.N]) == 0 and int(d.nb[d.N]) == spec.nx
    b = make_batch(0)
    x0 = b.fields["lb"][0][3:11]
    np.testing.assert_allclose(x0[:4], [0.2739, -0.4604, -0.9181, -0.9669], atol=1e-4)
    assert np.all(x0[4:] == 0.0)
    A, B = chain_dynamics(4, 0.5, (0, 1, 2))
    assert np.max(np.abs(np.linalg.eigvals(A))) <= 1 + 1e-12       # marginally stable
    assert B.shape == (8, 3)
    # per-QP seeds: batch rows equal single-QP draws
    b3 = make_batch(3, batch=2, N=4)
    s1 = make_batch(3, batch=1, start=1, N=4)
    assert np.array_equal(b3.fields["A"][1], s1.fields["A"][0])


def test_flop_closed_forms():
    # F_fac checks equal to the reference flop_counter
    assert rf.factor_flops(config_dim(CONFIGS[0])) == 58385
    assert rf.factor_flops(config_dim(CONFIGS[2])) == 2263158
    assert rf.factor_flops(config_dim(CONFIGS[3])) == 11243650
    assert rf.factor_flops(config_dim(CONFIGS[4])) == 153938600


def test_shard_ranges_cover_batch():
    for B in (0, 1, 7, 1024):
        for W in (1, 2, 3, 8):
            parts = [shard_range(B, r, W) for r in range(W)]
            assert parts[0][0] == 0 and parts[-1][1] == B
            assert all(parts[i][1] == parts[i + 1][0] for i in range(W - 1))
