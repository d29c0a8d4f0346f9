"""GPU vs CPU oracle for the modes beyond speed on random structure: the
team kernel's balance path (refinement, escapes) on every instantiated stage
shape with box subsets / one-sided rows / masks / general rows, and the
generic kernel (square-root, robust QR, speed_abs, balance) on random QPs with
soft rows.  The oracle is pinned to the reference for these modes
(tests/test_oracle_modes.py); rules as tests/modes_common.py."""

import numpy as np
import pytest

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200 import solver as S

from conftest import rel_err
from modes_common import mode_arg, solve_flops

pytestmark = pytest.mark.gpu


def host(rep):
    return {k: getattr(rep, k).cpu().numpy() for k in ("y", "pi", "lam", "t")} | {
        "status": rep.status_code.cpu().numpy(), "iters": rep.iterations.cpu().numpy(),
        "flops": rep.flops.cpu().numpy()}


def compare(got, ref, batch, arg, lam_tol=1e-8):
    for i in range(batch.B):
        if ref["status"][i] == 4:        # classical breakdown: rounding-borderline class
            assert got["status"][i] == 4
            continue
        assert got["status"][i] == ref["status"][i], i
        assert got["iters"][i] == ref["iters"][i], i
        df = int(got["flops"][i] - ref["flops"][i])
        if arg.itref_corr_max > 0:
            assert df % solve_flops(batch) == 0, df
        else:
            assert df == 0, df
        tol = 1e-2 if arg.abs_form else 1e-8
        for k in ("y", "pi", "t"):
            assert rel_err(got[k][i], ref[k][i]) <= tol, (k, i)
        assert rel_err(got["lam"][i], ref["lam"][i]) <= max(tol, lam_tol), ("lam", i)


@pytest.mark.parametrize("nx,nu,ng", [(8, 3, 0), (24, 4, 0), (30, 10, 10)])
@pytest.mark.parametrize("seed,N,nb", [(31, 6, 5), (32, 12, 200), (33, 3, 2)])
def test_team_kernel_balance_random_structure(cuda, oracle, nx, nu, ng, seed, N, nb):
    import qpgen

    # one structure (idxb, masks) for the batch; per-QP linear terms and offsets
    qps = []
    rng = np.random.default_rng(seed)
    for j in range(4):
        dims, stages, dyn = qpgen.random_ocp_fields(seed, N=N, nx=nx, nu=nu, nb=nb, ng=ng, ns=0,
                                                    inf_side=True, mask_last=True,
                                                    decay=0.9 / np.sqrt(nx))
        q = qpgen.build_qp(pkg, dims, stages, dyn)
        if j:
            for n in range(N + 1):
                q.set_field("q", n, q.get_field("q", n) + 0.3 * rng.standard_normal(nx))
                if n < N:
                    q.set_field("r", n, q.get_field("r", n) + 0.3 * rng.standard_normal(nu))
                    q.set_field("b", n, q.get_field("b", n) + 0.05 * rng.standard_normal(nx))
        qps.append(q)
    batch = OcpQpBatch.from_qps(qps)
    S._PLANS.clear()
    assert S.get_plan(batch).info()["kernel"] == "team"
    arg = mode_arg("balance6")
    got = host(solve_ocp_qp_batch(batch, arg))
    ref = oracle.solve(batch, arg, nthreads=4)
    compare(got, ref, batch, arg, lam_tol=1e-6 if ng else 1e-8)


@pytest.mark.parametrize("mode", ["balance6", "robust6", "sqrt8", "sqrtbal6", "abs8"])
@pytest.mark.parametrize("seed", [41, 42, 43])
def test_generic_kernel_modes_random_soft(cuda, oracle, mode, seed):
    import qpgen

    qps = [qpgen.build_qp(pkg, *qpgen.random_ocp_fields(seed * 10 + j, N=5 + j, nx=4, nu=2,
                                                         nb=4, ng=1, ns=2,
                                                         fix_x0=bool(j % 2)))
           for j in range(3)]
    arg = mode_arg(mode)
    for q in qps:   # different horizons: one plan per QP (generic kernel: soft rows)
        batch = OcpQpBatch.from_qps([q])
        got = host(solve_ocp_qp_batch(batch, arg))
        ref = oracle.solve(batch, arg, nthreads=1)
        compare(got, ref, batch, arg)
