"""GPU full condensing (csrc/ocpqp_condense.cu, full mode) + the dense-QP solve
on the fused IPM kernels + expand_solution, against the reference goldens
(tests/golden/fcond.npz) and the oracle.

Bar: condensed dense QP equal to the reference's condense() to 1e-12
relative; the dense solve takes the reference's status, iteration count and
counted flops, solution within 1e-8; the expanded OCP solution within 1e-8 of
the reference's expand_solution; whole config batches agree with the oracle.
"""

import os

import numpy as np
import pytest

import condense_oracle as co

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200.condensing import condense_batch, expand_batch
from paper_2003_02547_b200.generators import make_batch

from conftest import rel_err
from test_condense_oracle import source_qp
from test_fcond_oracle import fcond_cases, finite

pytestmark = pytest.mark.gpu

# dense field -> stage-0 field of the N = 0 form
DMAP = {"H": "R", "g": "r", "lb": "lb", "ub": "ub", "C": "D", "lg": "lg", "ug": "ug",
        "maskl": "maskl", "masku": "masku"}


@pytest.mark.parametrize("case", fcond_cases(), ids=lambda c: c[0])
def test_gpu_condense_solve_expand_matches_reference(cuda, speed_arg, golden, case):
    name, src, keep = case
    g = golden("fcond")
    batch = OcpQpBatch.from_qps([source_qp(src)])
    cb, cmap = condense_batch(batch, keep)
    nv, ne, nb, ng, ns, kept = (int(v) for v in g[f"{name}_dims"])
    assert cb.dim.N == 0 and list(cb.dim.nx) == [0]
    assert (cmap.nv, int(cb.dim.nb[0]), int(cb.dim.ng[0]), int(cmap.keep_x0)) == (nv, nb, ng, kept)
    q = cb.numpy().qp(0)
    assert np.array_equal(q.get_field("idxb", 0), g[f"{name}_idxb"])
    for f, o in DMAP.items():
        assert rel_err(finite(q.get_field(o, 0)).reshape(-1),
                       finite(g[f"{name}_{f}"]).reshape(-1)) <= 1e-12, f
    rep = solve_ocp_qp_batch(cb, speed_arg)
    assert int(rep.status_code.cpu()[0]) == int(g[f"{name}_dense_status"])
    assert int(rep.iterations.cpu()[0]) == int(g[f"{name}_dense_iters"])
    assert int(rep.flops.cpu()[0]) == int(g[f"{name}_dense_flops"])
    for k in ("y", "lam", "t"):
        assert rel_err(getattr(rep, k).cpu().numpy()[0], g[f"{name}_dense_{k}"]) <= 1e-8, k
    y, pi, lam, t = expand_batch(rep, cmap, batch)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v.cpu().numpy()[0], g[f"{name}_full_{k}"]) <= 1e-8, k


def test_gpu_expand_of_reference_dense_solution(cuda, golden):
    g = golden("fcond")
    for name, src, keep in fcond_cases():
        batch = OcpQpBatch.from_qps([source_qp(src)])
        _, cmap = condense_batch(batch, keep)
        dense = tuple(g[f"{name}_dense_{k}"][None] for k in ("y", "pi", "lam", "t"))
        y, pi, lam, t = expand_batch(dense, cmap, batch)
        for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
            assert rel_err(v.cpu().numpy()[0], g[f"{name}_full_{k}"]) <= 1e-12, (name, k)


def test_gpu_single_qp_dropins(cuda, golden):
    """condense / solve_dense_qp / expand_solution (the reference's calls)."""
    g = golden("fcond")
    name, src, keep = [c for c in fcond_cases() if c[0] == "c1"][0]
    qp = source_qp(src)
    arg = pkg.mode_preset("speed").with_tol(1e-8)
    dq, cmap = pkg.condense(qp)
    assert isinstance(dq, pkg.DenseQp) and dq.nv == cmap.nv and dq.ne == 0
    rep = pkg.solve_dense_qp(dq, arg)
    assert rep.iterations == int(g[f"{name}_dense_iters"])
    assert rel_err(rep.solution.v, g[f"{name}_dense_y"]) <= 1e-8
    full = pkg.expand_solution(rep.solution, cmap, qp)
    assert rel_err(full.y, g[f"{name}_full_y"]) <= 1e-8
    assert rel_err(full.pi, g[f"{name}_full_pi"]) <= 1e-8


@pytest.mark.parametrize("cfg,B", [(1, 1024), (2, 64), (3, 2)])
def test_gpu_condensed_config_batch_vs_oracle(cuda, oracle, speed_arg, cfg, B):
    """A BASELINE-config batch: GPU condensing equals the oracle's per QP; the
    GPU dense solve of the batch equals the C oracle's on the same dense QPs
    (status, iterations, flops, solutions); expansion equals the oracle's."""
    batch = make_batch(cfg, batch=B)
    cb, cmap = condense_batch(batch)
    host = cb.numpy()
    check = [0, B // 2, B - 1]
    qps = [batch.qp(i) for i in check]
    for j, i in enumerate(check):
        dense, _ = co.full_condense(qps[j])
        q = host.qp(i)
        for f, o in DMAP.items():
            assert rel_err(finite(q.get_field(o, 0)).reshape(-1),
                           finite(dense[f]).reshape(-1)) <= 1e-11, (i, f)
    rep = solve_ocp_qp_batch(cb, speed_arg)
    ref = oracle.solve(host, speed_arg, nthreads=os.cpu_count() or 4)
    assert np.array_equal(rep.status_code.cpu().numpy(), ref["status"])
    assert np.array_equal(rep.iterations.cpu().numpy(), ref["iters"])
    assert np.array_equal(rep.flops.cpu().numpy(), ref["flops"])
    ys = rep.y.cpu().numpy()
    errs = [rel_err(ys[i], ref["y"][i]) for i in range(B)]
    assert max(errs) <= 1e-8
    y, pi, lam, t = expand_batch(rep, cmap, batch)
    for j, i in enumerate(check):
        _, m = co.full_condense(qps[j])
        fy, fpi, flam, ft = co.full_expand(qps[j], m, ys[i], rep.lam.cpu().numpy()[i],
                                           rep.t.cpu().numpy()[i])
        for k, v, r in (("y", y, fy), ("pi", pi, fpi), ("lam", lam, flam), ("t", t, ft)):
            assert rel_err(v.cpu().numpy()[i], r) <= 1e-10, (i, k)


@pytest.mark.parametrize("case", fcond_cases(), ids=lambda c: c[0])
def test_gpu_square_root_condense_matches_reference(cuda, golden, case):
    """condense(variant="square_root") on the GPU (U_n = qr_cholesky([chol(Q_n)'; U_{n+1} A]),
    condensing.py:134-146) against the reference's dense H and g; the other
    fields do not depend on the cost recursion and must equal the classical ones."""
    name, src, keep = case
    g, gc = golden("fcond_sqrt"), golden("fcond")
    batch = OcpQpBatch.from_qps([source_qp(src)])
    cb, cmap = condense_batch(batch, keep, variant="square_root")
    q = cb.numpy().qp(0)
    assert rel_err(q.get_field("R", 0).reshape(-1), g[f"{name}_H"].reshape(-1)) <= 1e-12
    assert rel_err(q.get_field("r", 0).reshape(-1), g[f"{name}_g"].reshape(-1)) <= 1e-12
    for f, o in DMAP.items():
        if f not in ("H", "g"):
            assert rel_err(finite(q.get_field(o, 0)).reshape(-1),
                           finite(gc[f"{name}_{f}"]).reshape(-1)) <= 1e-12, f
    # the same plan goes back to the classical recursion
    cb2, _ = condense_batch(batch, keep)
    assert rel_err(cb2.numpy().qp(0).get_field("R", 0).reshape(-1), gc[f"{name}_H"].reshape(-1)) <= 1e-12


def test_gpu_square_root_condense_raises_like_the_reference(cuda, golden):
    from paper_2003_02547_b200.errors import NotPositiveDefinite

    assert int(golden("fcond_sqrt")["npd_raises"]) == 1
    qp = source_qp(fcond_cases()[0][1])
    qp.set_field("Q", 2, np.zeros((3, 3)))
    with pytest.raises(NotPositiveDefinite):
        pkg.condense(qp, variant="square_root")
    pkg.condense(qp)   # the classical recursion tolerates a semidefinite stage cost
    batch = OcpQpBatch.from_qps([source_qp(fcond_cases()[0][1]), qp])
    with pytest.raises(NotPositiveDefinite, match="QP 1"):
        condense_batch(batch, variant="square_root")
