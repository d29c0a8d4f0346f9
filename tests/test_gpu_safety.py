"""Race / out-of-bounds proxies for the shaped kernels (compute-sanitizer is
closed on this GPU pool: runs under it left GPUs needing a reset).

* Every QP is solved by one CTA with no cross-QP state, so a QP's result must
  be bit-identical whether it is solved alone, at another batch position,
  or again: any shared-memory race, missing barrier or TMA phase slip between
  the producer thread and the team shows up as a bitwise difference.
* Output buffers are placed inside NaN guard bands; the kernels must not
  write outside their [B, n] rows.
"""

import numpy as np
import pytest

from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
from paper_2003_02547_b200.generators import make_batch

pytestmark = pytest.mark.gpu

CASES = [(1, 64, None), (2, 8, None), (3, 8, None), (4, 4, None), (4, 3, 7)]


def _host(rep):
    return {k: getattr(rep, k).cpu().numpy() for k in ("y", "pi", "lam", "t", "res")} | {
        "iters": rep.iterations.cpu().numpy(), "status": rep.status_code.cpu().numpy()}


@pytest.mark.parametrize("cfg,B,N", CASES)
@pytest.mark.parametrize("mode", ["speed", "balance"])
def test_gpu_results_bitwise_stable(cuda, cfg, B, N, mode):
    arg = mode_preset(mode).with_tol(1e-8 if mode == "speed" else 1e-6)
    batch = make_batch(cfg, batch=B, N=N).to("cuda")
    runs = [_host(solve_ocp_qp_batch(batch, arg, trace=False)) for _ in range(3)]
    for r in runs[1:]:
        for k in runs[0]:
            assert np.array_equal(r[k], runs[0][k], equal_nan=True), k
    # the last QP solved alone and at the front of a reversed batch
    alone = _host(solve_ocp_qp_batch(make_batch(cfg, batch=1, start=B - 1, N=N), arg, trace=False))
    rev = _host(solve_ocp_qp_batch(make_batch(cfg, batch=B, N=N).select(list(range(B))[::-1]), arg,
                                   trace=False))
    for k in alone:
        assert np.array_equal(alone[k][0], runs[0][k][B - 1], equal_nan=True), k
        assert np.array_equal(rev[k][0], runs[0][k][B - 1], equal_nan=True), k


@pytest.mark.parametrize("cfg,B,N", [(1, 16, None), (4, 2, 9)])
def test_gpu_outputs_stay_inside_guard_bands(cuda, cfg, B, N):
    import torch

    arg = mode_preset("speed").with_tol(1e-8)
    batch = make_batch(cfg, batch=B, N=N).to("cuda")
    lay = batch.layout
    G = 64
    bufs, out = {}, {}
    for k, n, dt in (("y", lay.ny, torch.float64), ("pi", lay.ne, torch.float64),
                     ("lam", lay.nc, torch.float64), ("t", lay.nc, torch.float64),
                     ("res", 5, torch.float64), ("status", 1, torch.int32),
                     ("iters", 1, torch.int32), ("flops", 1, torch.int64)):
        fill = float("nan") if dt == torch.float64 else -7
        buf = torch.full((B * n + 2 * G,), fill, dtype=dt, device="cuda")
        bufs[k] = buf
        v = buf[G:G + B * n]
        out[k] = v.view(B, n) if k not in ("status", "iters", "flops") else v
    out["trace"] = None
    rep = solve_ocp_qp_batch(batch, arg, trace=False, out=out)
    ref = _host(solve_ocp_qp_batch(batch, arg, trace=False))
    for k, buf in bufs.items():
        h = buf.cpu().numpy()
        if h.dtype == np.float64:
            assert np.all(np.isnan(h[:G])) and np.all(np.isnan(h[-G:])), k
        else:
            assert np.all(h[:G] == -7) and np.all(h[-G:] == -7), k
    assert np.array_equal(rep.y.cpu().numpy(), ref["y"])
    assert np.array_equal(rep.iterations.cpu().numpy(), ref["iters"])


def test_dispatch_hint_changes_nothing_but_the_order(cuda):
    """ocpqp_plan_dispatch_hint (opt-in): the QPs of a solve are handed out in
    the order of the plan's previous solve's iteration counts, the slowest to
    the CTAs alone on their SM.  Results, iteration counts, statuses and flop
    counts must be bit-identical with and without it, on the full config-4
    batch (256 CTAs, two per SM: the case the hint is for) and on a batch that
    runs in several waves."""
    import torch

    from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.solver import get_plan

    arg = mode_preset("speed").with_tol(1e-8)
    for cfg, B in ((4, 256), (3, 512)):
        dev = make_batch(cfg, batch=B).to("cuda")
        base = solve_ocp_qp_batch(dev, arg, trace=False)
        ref = {k: getattr(base, k).clone() for k in ("y", "pi", "lam", "t", "iterations", "status_code", "flops")}
        plan = get_plan(dev)
        plan.dispatch_hint(True)
        try:
            for _ in range(3):   # the first hinted solve only records the counts
                rep = solve_ocp_qp_batch(dev, arg, trace=False)
                torch.cuda.synchronize()
                for k, v in ref.items():
                    assert torch.equal(getattr(rep, k), v), (cfg, k)
        finally:
            plan.dispatch_hint(False)
        rep = solve_ocp_qp_batch(dev, arg, trace=False)
        for k, v in ref.items():
            assert torch.equal(getattr(rep, k), v), (cfg, k)
