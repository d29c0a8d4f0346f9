"""Pin the CPU oracle's modes beyond speed -- balance / robust (iterative
refinement, QR array algorithm, fallback ladder), the square-root Riccati
variant and the absolute formulation (speed_abs) -- to the real reference's
outputs in tests/golden/modes.npz (see tests/modes_common.py for the rules)."""

import pytest

from modes_common import HEAVY, MODE_NAMES, SOURCES, check_mode_solve, mode_arg, source_batch

from conftest import STATUS

pytestmark = pytest.mark.filterwarnings("ignore")


@pytest.mark.parametrize("mode", MODE_NAMES)
@pytest.mark.parametrize("src", SOURCES)
def test_oracle_mode_matches_reference(oracle, golden, src, mode):
    g = golden("modes")
    batch = source_batch(src)
    out = oracle.solve(batch, mode_arg(mode), nthreads=1)
    check_mode_solve(out, 0, g, f"{src}_{mode}", mode, batch)


@pytest.mark.parametrize("src,mode", [(s, m) for s, ms in HEAVY for m in ms])
def test_oracle_mode_config4(oracle, golden, src, mode):
    g = golden("modes")
    batch = source_batch(src)
    out = oracle.solve(batch, mode_arg(mode), nthreads=1)
    check_mode_solve(out, 0, g, f"{src}_{mode}", mode, batch)


@pytest.mark.parametrize("mode", MODE_NAMES)
def test_oracle_mode_failure_ladder(oracle, golden, mode):
    """Indefinite scalar LQR: every rung of _factor_with_policy fails; the
    flop count pins which rungs ran (classical, per-stage QR, whole QR,
    regularised retry -- solver.py:145-164, kkt_ocp.py:180-191)."""
    import qpgen

    import paper_2003_02547_b200 as pkg
    from paper_2003_02547_b200 import OcpQpBatch

    g = golden("modes")
    q = qpgen.scalar_lqr(pkg)
    q.set_field("r", 0, [1.0])
    q.set_field("R", 0, [[-1.0]])
    q.set_field("Q", 0, [[-1.0]])
    q.set_field("Q", 1, [[-1.0]])
    out = oracle.solve(OcpQpBatch.from_qps([q]), mode_arg(mode), nthreads=1)
    assert int(out["status"][0]) == int(g[f"indef_{mode}_status"])
    assert int(out["iters"][0]) == int(g[f"indef_{mode}_iters"])
    assert int(out["flops"][0]) == int(g[f"indef_{mode}_flops"])


@pytest.mark.parametrize("mode", MODE_NAMES)
def test_oracle_mode_rank_deficient(oracle, golden, mode):
    """Robust mode meets a rank-deficient QR stack: the reference raises
    RankDeficient out of the solve; the oracle reports status 7."""
    import qpgen

    import paper_2003_02547_b200 as pkg
    from paper_2003_02547_b200 import OcpQpBatch

    g = golden("modes")
    batch = OcpQpBatch.from_qps([qpgen.rank_deficient(pkg)])
    out = oracle.solve(batch, mode_arg(mode), nthreads=1)
    if int(g[f"rankdef_{mode}_raised"]):
        assert int(out["status"][0]) == 7
    else:
        check_mode_solve(out, 0, g, f"rankdef_{mode}", mode, batch)
    assert STATUS["Success"] == 0
