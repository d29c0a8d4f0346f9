"""Pin the CPU oracle (oracle/ocpqp_oracle.c) to the real reference's outputs.

The fixtures were produced by tests/golden/make_golden.py importing the
reference package (/root/reference/pkg/src/mpcqp).  A green run here is what
makes the oracle trustworthy as the GPU path's checker.
"""

import numpy as np
import pytest

from conftest import cfg_cases, random_case_qp, random_cases, rel_err

from paper_2003_02547_b200 import OcpQpBatch
from paper_2003_02547_b200.generators import make_batch

pytestmark = pytest.mark.filterwarnings("ignore")


def _check_solve(out, i, g, prefix, sol_tol=1e-9):
    assert int(out["status"][i]) == int(g[f"{prefix}_status"])
    assert int(out["iters"][i]) == int(g[f"{prefix}_iters"])
    assert int(out["flops"][i]) == int(g[f"{prefix}_flops"])
    for k in ("y", "pi", "lam", "t"):
        assert rel_err(out[k][i], g[f"{prefix}_{k}"]) <= sol_tol, k
    res = g[f"{prefix}_res"]
    assert np.all(np.abs(out["res"][i] - res) <= 1e-8 * np.maximum(1.0, np.abs(res)))
    tr = g[f"{prefix}_trace"]
    it = int(g[f"{prefix}_iters"])
    np.testing.assert_allclose(out["trace"][i, :it, :4], tr[:, :4], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("cfg,indices,N", cfg_cases())
def test_oracle_matches_reference_on_configs(oracle, speed_arg, golden, cfg, indices, N):
    g = golden("solve_cfg")
    batch = make_batch(cfg, batch=max(indices) + 1, N=N).select(indices)
    out = oracle.solve(batch, speed_arg, nthreads=4)
    for j, i in enumerate(indices):
        _check_solve(out, j, g, f"c{cfg}_q{i}", sol_tol=1e-9 if cfg != 3 else 1e-8)


@pytest.mark.parametrize("case", random_cases(), ids=lambda c: f"seed{c[0]}")
def test_oracle_matches_reference_random(oracle, speed_arg, golden, case):
    seed, kw = case
    g = golden("solve_random")
    batch = OcpQpBatch.from_qps([random_case_qp(seed, kw)])
    out = oracle.solve(batch, speed_arg, nthreads=1)
    _check_solve(out, 0, g, f"s{seed}")


@pytest.mark.parametrize("case", random_cases(), ids=lambda c: f"seed{c[0]}")
def test_oracle_newton_step_matches_reference(oracle, golden, case):
    seed, kw = case
    g = golden("newton")
    p = f"s{seed}"
    batch = OcpQpBatch.from_qps([random_case_qp(seed, kw)])
    out = oracle.newton_step(batch, g[f"{p}_lam"], g[f"{p}_t"], g[f"{p}_r_g"], g[f"{p}_r_b"],
                             g[f"{p}_r_d"], g[f"{p}_r_m"], want_P=True)
    assert int(out["fail"][0]) == -1
    ref = np.concatenate([g[f"{p}_{k}"] for k in ("dy", "dpi", "dlam", "dt")])
    got = np.concatenate([out[k][0] for k in ("dy", "dpi", "dlam", "dt")])
    assert rel_err(got, ref) <= 1e-10
    assert rel_err(out["P"][0], g[f"{p}_P"]) <= 1e-12


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_oracle_newton_step_config_shapes(oracle, golden, cfg):
    g = golden("newton")
    p = f"c{cfg}"
    batch = make_batch(cfg, batch=8).select([7])
    out = oracle.newton_step(batch, g[f"{p}_lam"], g[f"{p}_t"], g[f"{p}_r_g"], g[f"{p}_r_b"],
                             g[f"{p}_r_d"], g[f"{p}_r_m"])
    ref = np.concatenate([g[f"{p}_{k}"] for k in ("dy", "dpi", "dlam", "dt")])
    got = np.concatenate([out[k][0] for k in ("dy", "dpi", "dlam", "dt")])
    assert rel_err(got, ref) <= 1e-9


@pytest.mark.parametrize("case", random_cases(), ids=lambda c: f"seed{c[0]}")
def test_oracle_residuals_match_reference(oracle, golden, case):
    seed, kw = case
    g = golden("residuals")
    p = f"s{seed}"
    batch = OcpQpBatch.from_qps([random_case_qp(seed, kw)])
    out = oracle.residuals(batch, g[f"{p}_y"], g[f"{p}_pi"], g[f"{p}_lam"], g[f"{p}_t"])
    for k in ("r_g", "r_b", "r_d", "r_m"):
        assert rel_err(out[k][0], g[f"{p}_{k}"]) <= 1e-13, k
    np.testing.assert_allclose(out["norms"][0], g[f"{p}_norms"], rtol=1e-12, atol=1e-14)


def test_oracle_known_answers(oracle, speed_arg, golden):
    import qpgen

    import paper_2003_02547_b200 as pkg

    k = golden("known")
    # scalar LQR: P1 = 1, P0 = 1.5 (reference test_kkt_ocp.py:37-43)
    b = OcpQpBatch.from_qps([qpgen.scalar_lqr(pkg)])
    nc = b.layout.nc
    out = oracle.newton_step(b, np.zeros(nc), np.zeros(nc), np.zeros(b.layout.ny),
                             np.zeros(b.layout.ne), np.zeros(nc), np.zeros(nc), want_P=True)
    assert abs(out["P"][0][1] - float(k["lqr_P1"])) <= 1e-12
    assert abs(out["P"][0][0] - float(k["lqr_P0"])) <= 1e-12
    # bounded scalar LQR: u0 = -1.5 (reference test_solver.py:100-116)
    out = oracle.solve(OcpQpBatch.from_qps([qpgen.scalar_lqr(pkg, bounds=True)]), speed_arg)
    assert int(out["status"][0]) == int(k["lqr_bounds_status"]) == 0
    assert abs(out["y"][0][0] - float(k["lqr_bounds_u0"])) <= 1e-8
    # indefinite input weight -> Failure, with the reference's flop count
    q = qpgen.scalar_lqr(pkg)
    q.set_field("r", 0, [1.0])
    q.set_field("R", 0, [[-1.0]])
    q.set_field("Q", 0, [[-1.0]])
    q.set_field("Q", 1, [[-1.0]])
    out = oracle.solve(OcpQpBatch.from_qps([q]), speed_arg)
    assert int(out["status"][0]) == int(k["indef_status"]) == 4
    assert int(out["iters"][0]) == int(k["indef_iters"])
    assert int(out["flops"][0]) == int(k["indef_flops"])
    # crossed bounds -> never Success
    q = qpgen.scalar_lqr(pkg, bounds=True)
    q.set_field("lb", 1, [1.0])
    q.set_field("ub", 1, [0.0])
    out = oracle.solve(OcpQpBatch.from_qps([q]), speed_arg)
    assert int(out["status"][0]) == int(k["infeas_status"])
    assert int(out["iters"][0]) == int(k["infeas_iters"])
