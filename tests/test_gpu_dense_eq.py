"""Dense QPs with equality constraints on the GPU (csrc/ocpqp_dense.cu) against
the reference's solve_dense_qp (tests/golden/dense_eq.npz, made by
tests/golden/make_golden.py dense_eq): the Schur-complement and null-space
methods of kkt_dense.py:117-231 in speed mode, including an exactly singular
equality block (Failure after the regularised retry, same counted flops).

Bar: status, iteration count and counted flops identical; v / pi / lam / t
within 1e-8 relative; final residual norms |d| <= 1e-8 max(1, |ref|)."""

from dataclasses import replace

import numpy as np
import pytest

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200.dense import solve_dense_qp, solve_dense_qp_batch

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu


def cases():
    src = (GOLDEN / "make_golden.py").read_text()
    start = src.index("DENSE_EQ_CASES = [")
    end = src.index("]\n", start) + 1
    ns = {}
    exec(src[start:end], {}, ns)
    return ns["DENSE_EQ_CASES"]


def build(seed, nv, ne, nb, ng, rd):
    import sys

    sys.path.insert(0, str(GOLDEN))
    src = (GOLDEN / "make_golden.py").read_text()
    i0 = src.index("def dense_eq_qp(")
    i1 = src.index("\ndef dense_eq():")
    ns = {"np": np}
    exec(src[i0:i1], ns)
    return ns["dense_eq_qp"](pkg, seed, nv, ne, nb, ng, rd)


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"e{c[0]}-{c[5]}")
def test_gpu_dense_eq_matches_reference(cuda, golden, case):
    seed, nv, ne, nb, ng, method, rd = case
    g = golden("dense_eq")
    p = f"e{seed}"
    q = build(seed, nv, ne, nb, ng, rd)
    arg = replace(pkg.mode_preset("speed").with_tol(1e-8), kkt_method=method)
    rep = solve_dense_qp(q, arg)
    from paper_2003_02547_b200.ipm import STATUS_CODES

    assert rep.stats.status is STATUS_CODES[int(g[f"{p}_status"])]
    assert rep.iterations == int(g[f"{p}_iters"])
    assert rep.stats.flops == int(g[f"{p}_flops"])
    if int(g[f"{p}_status"]) != 0:
        return
    s = rep.solution
    for k, v in (("y", s.y), ("pi", s.pi), ("lam", s.lam), ("t", s.t)):
        assert rel_err(v, g[f"{p}_{k}"]) <= 1e-8, k
    r = np.array([rep.stats.res_g, rep.stats.res_b, rep.stats.res_d, rep.stats.res_m, rep.stats.mu])
    ref = g[f"{p}_res"]
    assert np.all(np.abs(r - ref) <= 1e-8 * np.maximum(1.0, np.abs(ref)))
    assert rep.residuals.max_norm() <= 1e-8
    it = int(g[f"{p}_iters"])
    tr = np.array([[x.alpha_aff, x.alpha, x.mu, x.sigma] for x in rep.stats.trace])
    np.testing.assert_allclose(tr, g[f"{p}_trace"][:it, :4], rtol=1e-6, atol=1e-12)


def test_gpu_dense_eq_batch_equals_single(cuda):
    """A batch of dense QPs (same structure) equals the one-by-one solves."""
    qs = []
    for k in range(3):   # one structure (idxb), different costs
        q = build(62, 12, 4, 6, 3, False)
        q.set_field("g", np.random.default_rng(k).standard_normal(12))
        qs.append(q)
    arg = pkg.mode_preset("speed").with_tol(1e-8)
    out = solve_dense_qp_batch(qs, arg)
    for i, q in enumerate(qs):
        r = solve_dense_qp(q, arg)
        assert np.array_equal(out["y"].cpu().numpy()[i], r.solution.y)
        assert int(out["iters"].cpu()[i]) == r.iterations


def test_dense_eq_unsupported_modes_raise(cuda):
    q = build(61, 8, 2, 4, 2, False)
    with pytest.raises(NotImplementedError):
        solve_dense_qp(q, pkg.mode_preset("balance").with_tol(1e-6))
