"""Pin the closed-loop MPC checker (oracle/mpc_oracle.py) to the reference's
run_closed_loop trajectories and _shift_guess (tests/golden/closed_loop.npz)."""

import numpy as np
import pytest

from conftest import rel_err

CASES = [
    ("m3", dict(masses=3, horizon=10), 8, "balance", 1e-6, "primal_dual"),
    ("m4", dict(masses=4, horizon=15, x0=[0.5, -0.3, 0.2, -0.6, 0.0, 0.0, 0.0, 0.0]), 6,
     "speed", 1e-8, "primal_dual"),
    ("m2", dict(masses=2, horizon=10), 5, "speed", 1e-8, "primal"),
]


def test_shift_guess_matches_reference(oracle, golden):
    import mpc_oracle

    from paper_2003_02547_b200 import OcpQpBatch
    from paper_2003_02547_b200.mpc import MassSpringConfig, gen_mass_spring

    g = golden("closed_loop")
    batch = OcpQpBatch.from_qps([gen_mass_spring(MassSpringConfig(masses=3, horizon=10))])
    got = mpc_oracle.shift_guess(batch, tuple(g[f"shift_sol_{k}"] for k in ("y", "pi", "lam", "t")))
    for k, a in zip(("y", "pi", "lam", "t"), got):
        assert rel_err(a, g[f"shift_guess_{k}"]) <= 1e-12, k


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_closed_loop_matches_reference(oracle, golden, case):
    import mpc_oracle

    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.mpc import MassSpringConfig

    name, kw, steps, preset, tol, warm = case
    g = golden("closed_loop")
    out = mpc_oracle.run_closed_loop(MassSpringConfig(**kw), steps,
                                     mode_preset(preset).with_tol(tol), warm, compare_cold=True)
    np.testing.assert_array_equal(out["status"], g[f"{name}_status"])
    np.testing.assert_array_equal(out["iters"], g[f"{name}_iters"])
    np.testing.assert_array_equal(out["cold_iters"], g[f"{name}_cold_iters"])
    assert rel_err(out["states"], g[f"{name}_states"]) <= 1e-8
    assert rel_err(out["inputs"], g[f"{name}_inputs"]) <= 1e-8
