"""GPU closed-loop MPC: the device shift kernel (ocpqp_shift_guess) and the
batched closed-loop driver against the reference's trajectories
(tests/golden/closed_loop.npz) and against the CPU checker (oracle/mpc_oracle.py)."""

import numpy as np
import pytest

from conftest import rel_err

from test_mpc_oracle import CASES

pytestmark = pytest.mark.gpu


def test_gpu_shift_matches_reference(cuda, golden):
    import torch

    from paper_2003_02547_b200 import OcpQpBatch
    from paper_2003_02547_b200.mpc import MassSpringConfig, gen_mass_spring, shift_guess

    g = golden("closed_loop")
    batch = OcpQpBatch.from_qps([gen_mass_spring(MassSpringConfig(masses=3, horizon=10))])
    dev = batch.to("cuda")
    sol = tuple(torch.as_tensor(g[f"shift_sol_{k}"][None], dtype=torch.float64, device="cuda")
                for k in ("y", "pi", "lam", "t"))
    got = shift_guess(dev, sol)
    for k, a in zip(("y", "pi", "lam", "t"), got):
        assert rel_err(a.cpu().numpy()[0], g[f"shift_guess_{k}"]) <= 1e-12, k


def test_gpu_shift_batch_vs_oracle(cuda, oracle):
    """Shift every solution of a solved config-1 batch; compare with the numpy
    restatement per QP."""
    import mpc_oracle

    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.mpc import shift_guess

    batch = make_batch(1, batch=64)
    dev = batch.to("cuda")
    rep = solve_ocp_qp_batch(dev, mode_preset("speed").with_tol(1e-8))
    got = [a.cpu().numpy() for a in shift_guess(dev, (rep.y, rep.pi, rep.lam, rep.t))]
    sol = [a.cpu().numpy() for a in (rep.y, rep.pi, rep.lam, rep.t)]
    for i in range(0, 64, 7):
        one = batch.select([i])
        ref = mpc_oracle.shift_guess(one, tuple(s[i] for s in sol))
        for a, r in zip(got, ref):
            assert rel_err(a[i], r) <= 1e-12


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_gpu_closed_loop_matches_reference(cuda, golden, case):
    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.mpc import MassSpringConfig, run_closed_loop

    name, kw, steps, preset, tol, warm = case
    g = golden("closed_loop")
    res = run_closed_loop(MassSpringConfig(**kw), steps, arg=mode_preset(preset).with_tol(tol),
                          warm_start=warm, compare_cold=True)
    assert [r.iterations for r in res.records] == list(g[f"{name}_iters"])
    assert [r.cold_iterations for r in res.records] == list(g[f"{name}_cold_iters"])
    assert all(r.status == "Success" for r in res.records)
    assert rel_err(res.states, g[f"{name}_states"]) <= 1e-8
    assert rel_err(res.inputs, g[f"{name}_inputs"]) <= 1e-8


def test_gpu_closed_loop_batch_vs_oracle(cuda, oracle):
    """64 plants in lockstep (balance mode, the reference default) against the
    CPU checker run plant by plant."""
    import mpc_oracle

    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.mpc import MassSpringConfig, run_closed_loop_batch

    rng = np.random.default_rng(5)
    cfg = MassSpringConfig(masses=4, horizon=12)
    x0s = np.concatenate([rng.uniform(-1.0, 1.0, (64, 4)), np.zeros((64, 4))], axis=1)
    arg = mode_preset("balance").with_tol(1e-6)
    res = run_closed_loop_batch(cfg, x0s, 6, arg=arg)
    for i in (0, 17, 63):
        ref = mpc_oracle.run_closed_loop(MassSpringConfig(masses=4, horizon=12, x0=x0s[i]), 6, arg)
        assert [r.iterations for r in res[i].records] == list(ref["iters"])
        assert rel_err(res[i].states, ref["states"]) <= 1e-8
