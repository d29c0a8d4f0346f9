"""Full condensing + the dense-QP solve: oracle and host API vs the reference.

tests/golden/fcond.npz holds, per case, the reference's condense() output
(condensing.py:160-340), its solve_dense_qp report (solver.py:98-100) and
expand_solution (condensing.py:343-429) of that solution, plus the direct
solve's iteration count.  The oracle (oracle/condense_oracle.py full_condense
/ full_expand; the C oracle on the N = 0 form for the IPM) is pinned here; the
GPU path is checked against both in test_gpu_fcond.py.
"""

import numpy as np
import pytest

import condense_oracle as co

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import DenseQp, OcpQpBatch, dense_to_ocp, ocp_to_dense
from paper_2003_02547_b200.condensing import detect_fixed_x0
from paper_2003_02547_b200.errors import CondenseError, DimensionMismatch, IndexOutOfRange
from paper_2003_02547_b200.layout import OcpLayout

from conftest import GOLDEN, rel_err
from test_condense_oracle import source_qp

DFIELDS = ("H", "g", "lb", "ub", "C", "lg", "ug", "maskl", "masku")


def fcond_cases():
    src = (GOLDEN / "make_golden.py").read_text()
    start = src.index("FCOND_CASES = [")
    end = src.index("]\n", start) + 1
    ns = {}
    exec(src[start:end], {"dict": dict, "True": True, "None": None}, ns)
    return ns["FCOND_CASES"]


def finite(a):
    return np.nan_to_num(np.asarray(a, dtype=float), posinf=1e300, neginf=-1e300)


def golden_dense(g, name):
    nv, ne, nb, ng, ns, _ = (int(v) for v in g[f"{name}_dims"])
    dq = DenseQp(nv, ne, nb, ng, ns)
    for f in DFIELDS + ("idxb",):
        dq.set_field(f, g[f"{name}_{f}"])
    return dq


@pytest.mark.parametrize("case", fcond_cases(), ids=lambda c: c[0])
def test_oracle_full_condense_matches_reference(golden, case):
    name, src, keep = case
    g = golden("fcond")
    dense, cmap = co.full_condense(source_qp(src), keep)
    nv, ne, nb, ng, ns, kept = (int(v) for v in g[f"{name}_dims"])
    assert (len(dense["g"]), len(dense["idxb"]), len(dense["lg"]), int(cmap["keep_x0"])) == \
        (nv, nb, ng, kept)
    assert np.array_equal(dense["idxb"], g[f"{name}_idxb"])
    for f in DFIELDS:
        assert rel_err(finite(dense[f]).reshape(-1), finite(g[f"{name}_{f}"]).reshape(-1)) <= 1e-12, f


@pytest.mark.parametrize("case", fcond_cases(), ids=lambda c: c[0])
def test_oracle_dense_solve_is_the_n0_ocp_solve(golden, oracle, speed_arg, case):
    """The reference's dense backend == the IPM on the N = 0 form (same flops)."""
    name = case[0]
    g = golden("fcond")
    b = OcpQpBatch.from_qps([dense_to_ocp(golden_dense(g, name))])
    ref = oracle.solve(b, speed_arg, nthreads=1)
    assert int(ref["status"][0]) == int(g[f"{name}_dense_status"])
    assert int(ref["iters"][0]) == int(g[f"{name}_dense_iters"])
    assert int(ref["flops"][0]) == int(g[f"{name}_dense_flops"])
    for k in ("y", "lam", "t"):
        assert rel_err(ref[k][0], g[f"{name}_dense_{k}"]) <= 1e-8, k


@pytest.mark.parametrize("case", fcond_cases(), ids=lambda c: c[0])
def test_oracle_expand_solution_matches_reference(golden, case):
    name, src, keep = case
    g = golden("fcond")
    qp = source_qp(src)
    _, cmap = co.full_condense(qp, keep)
    y, pi, lam, t = co.full_expand(qp, cmap, g[f"{name}_dense_y"], g[f"{name}_dense_lam"],
                                   g[f"{name}_dense_t"])
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v, g[f"{name}_full_{k}"]) <= 1e-10, k
    # the condensed route reaches the direct solution
    assert rel_err(y, g[f"{name}_direct_y"]) <= 1e-5


def test_dense_qp_object_and_n0_form():
    dq = DenseQp(3, 0, 2, 1, 1)
    assert dq.kind == "dense" and dq.get_field("idxb").tolist() == [0, 1]
    dq.set_field("H", np.eye(3) * 2.0)
    dq.set_field("C", np.ones((1, 3)))
    dq.set_field("lb", [-1.0, -2.0])
    with pytest.raises(DimensionMismatch):
        dq.set_field("g", np.zeros(2))
    with pytest.raises(IndexOutOfRange):
        dq.get_field("H", 0)
    with pytest.raises(pkg.UnknownField):
        dq.get_field("Q")
    with pytest.raises(pkg.InvalidDim):
        DenseQp(2, nb=3)
    q = dense_to_ocp(dq)
    assert q.dim.N == 0 and list(q.dim.nx) == [0] and list(q.dim.nu) == [3]
    assert np.array_equal(q.get_field("R", 0), dq.get_field("H"))
    back = ocp_to_dense(q)
    for f in ("H", "g", "C", "lb", "ub", "idxb", "maskl"):
        assert np.array_equal(back.get_field(f), dq.get_field(f))
    with pytest.raises(NotImplementedError):
        dense_to_ocp(DenseQp(2, ne=1))


def test_detect_fixed_x0_batch_rules():
    import qpgen

    qp = qpgen.build_qp(pkg, *qpgen.random_ocp_fields(21, N=3, nx=3, nu=2, nb=4, ng=1, ns=0,
                                                     fix_x0=True))
    all_fixed, rows = detect_fixed_x0(OcpQpBatch.from_qps([qp]))
    ref_fixed, _, ref_rows = co.detect_fixed_x0(qp)
    assert all_fixed == ref_fixed and rows == ref_rows
    q2 = qpgen.build_qp(pkg, *qpgen.random_ocp_fields(21, N=3, nx=3, nu=2, nb=4, ng=1, ns=0,
                                                     fix_x0=True))
    ub = q2.get_field("ub", 0)
    ub[rows[0][0]] += 1.0
    q2.set_field("ub", 0, ub)
    with pytest.raises(CondenseError):
        detect_fixed_x0(OcpQpBatch.from_qps([qp, q2]))
    assert detect_fixed_x0(OcpQpBatch.from_qps([q2]))[0] is False


@pytest.mark.parametrize("case", fcond_cases(), ids=lambda c: c[0])
def test_oracle_square_root_condense_matches_reference(golden, case):
    """condense(variant="square_root") (condensing.py:134-146): the oracle's restatement
    against the reference's H and g (fcond_sqrt.npz)."""
    name, src, keep = case
    g = golden("fcond_sqrt")
    dense, _ = co.full_condense(source_qp(src), keep, variant="square_root")
    for f in ("H", "g"):
        assert rel_err(dense[f].reshape(-1), g[f"{name}_{f}"].reshape(-1)) <= 1e-12, f


def test_oracle_square_root_condense_needs_definite_q(golden):
    assert int(golden("fcond_sqrt")["npd_raises"]) == 1
    qp = source_qp(fcond_cases()[0][1])
    qp.set_field("Q", 2, np.zeros((3, 3)))
    with pytest.raises(np.linalg.LinAlgError):
        co.full_condense(qp, variant="square_root")
    co.full_condense(qp)   # the classical recursion tolerates it
