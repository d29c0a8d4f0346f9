"""GPU partial condensing / expansion (csrc/ocpqp_condense.cu) vs the reference.

Bar: condensed QP fields equal the reference's partial_condense output to
1e-12 relative; the condensed QP solved on the GPU takes the reference's
iteration count; the expanded full-horizon solution matches the reference's
partial_expand within 1e-8 relative; config 4 direct vs condensed agree.
"""

import numpy as np
import pytest

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200.condensing import partial_condense_batch, partial_expand_batch
from paper_2003_02547_b200.generators import make_batch

from conftest import rel_err
from test_condense_oracle import FIELDS, pcond_cases, source_qp

pytestmark = pytest.mark.gpu


def finite(a):
    return np.nan_to_num(np.asarray(a), posinf=1e300, neginf=-1e300)


@pytest.mark.parametrize("case", pcond_cases(), ids=lambda c: c[0])
def test_gpu_partial_condense_matches_reference(cuda, speed_arg, golden, case):
    name, src, N1 = case
    g = golden("pcond")
    qp = source_qp(src)
    batch = OcpQpBatch.from_qps([qp])
    cb, pmap = partial_condense_batch(batch, N1)
    host = cb.numpy()
    dims = g[f"{name}_dims"]
    assert cb.dim.N == dims.shape[1] - 1
    assert list(cb.dim.nu) == list(dims[1]) and list(cb.dim.ng) == list(dims[3])
    q2 = host.qp(0)
    for k in range(cb.dim.N + 1):
        assert np.array_equal(q2.get_field("idxb", k), g[f"{name}_s{k}_idxb"])
        for f in FIELDS:
            assert rel_err(finite(q2.get_field(f, k)), finite(g[f"{name}_s{k}_{f}"])) <= 1e-12, (k, f)
        if k < cb.dim.N:
            for f in ("A", "B", "b"):
                assert rel_err(q2.get_field(f, k), g[f"{name}_s{k}_{f}"]) <= 1e-12, (k, f)
    # solve the condensed QP on the GPU, expand, compare with the reference
    rep = solve_ocp_qp_batch(cb, speed_arg)
    assert int(rep.status_code.cpu()[0]) == int(g[f"{name}_short_status"])
    assert int(rep.iterations.cpu()[0]) == int(g[f"{name}_short_iters"])
    y, pi, lam, t = partial_expand_batch(rep, pmap, batch)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v.cpu().numpy()[0], g[f"{name}_full_{k}"]) <= 1e-8, k


def test_gpu_partial_expand_of_reference_solution(cuda, golden):
    """Expansion alone, fed the reference's own condensed solution."""
    for name, src, N1 in pcond_cases():
        g = golden("pcond")
        batch = OcpQpBatch.from_qps([source_qp(src)])
        _, pmap = partial_condense_batch(batch, N1)
        short = tuple(g[f"{name}_short_{k}"][None] for k in ("y", "pi", "lam", "t"))
        y, pi, lam, t = partial_expand_batch(short, pmap, batch)
        for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
            assert rel_err(v.cpu().numpy()[0], g[f"{name}_full_{k}"]) <= 1e-12, (name, k)


def test_gpu_block_size_one_is_identity(cuda):
    batch = make_batch(1, batch=3)
    cb, _ = partial_condense_batch(batch, 1)
    src = batch.numpy()
    out = cb.numpy()
    for name in ("A", "B", "Q", "R", "lb", "ub"):
        a = np.broadcast_to(src.fields[name], out.fields[name].shape)
        assert np.array_equal(out.fields[name], a), name


def test_gpu_config4_condensed_vs_direct(cuda, oracle, speed_arg):
    """Config 4 (N=100 -> 20 blocks): condensed solve + expansion agrees with
    the direct solve; condensed iterations match the oracle on the condensed QP."""
    batch = make_batch(4, batch=2)
    direct = solve_ocp_qp_batch(batch, speed_arg)
    cb, pmap = partial_condense_batch(batch, 5)
    assert cb.dim.N == 20 and int(cb.dim.nu[0]) == 100
    assert int(cb.dim.nb[0]) == 160 and int(cb.dim.ng[0]) == 240
    rep = solve_ocp_qp_batch(cb, speed_arg)
    ref = oracle.solve(cb.numpy(), speed_arg)
    assert np.array_equal(rep.iterations.cpu().numpy(), ref["iters"])
    assert np.array_equal(rep.status_code.cpu().numpy(), ref["status"])
    y, pi, lam, t = partial_expand_batch(rep, pmap, batch)
    for i in range(2):
        assert rel_err(y.cpu().numpy()[i], direct.y.cpu().numpy()[i]) <= 1e-6


def test_gpu_config4_partial_path_full_size_matches_oracle(cuda, oracle, speed_arg):
    """BASELINE config 4's second way at full size (N = 100 -> N2 = 20 blocks of
    5 stages, nx = 60, nu = 20) on 32 QPs: the GPU's partial_condense_batch ->
    solve -> partial_expand_batch against the oracle's own partial path
    (oracle/condense_oracle.py restatement of condensing.py:451-619 + the C
    oracle solve of the condensed QP): condensed fields to 1e-12, identical
    status and iteration counts, expanded y / pi / lam / t within 1e-8
    relative, final residual norms as in test_gpu_parity.assert_res_parity."""
    import condense_oracle as co
    from paper_2003_02547_b200.layout import OcpLayout

    from test_gpu_parity import assert_res_parity

    n = 32
    batch = make_batch(4, batch=n)
    cb, pmap = partial_condense_batch(batch, 5)
    qps = [batch.qp(i) for i in range(n)]
    cq = [co.partial_condensed_qp(q, 5) for q in qps]
    ocb = OcpQpBatch.from_qps([c[0] for c in cq])
    assert ocb.dim.key() == cb.dim.key()
    got_c = cb.numpy()
    for i in (0, 17, 31):
        a, r = got_c.qp(i), ocb.qp(i)
        for k in range(cb.dim.N + 1):
            for f in FIELDS + (("A", "B", "b") if k < cb.dim.N else ()):
                assert rel_err(finite(a.get_field(f, k)), finite(r.get_field(f, k))) <= 1e-12, (i, k, f)
    rep = solve_ocp_qp_batch(cb, speed_arg)
    ref = oracle.solve(ocb, speed_arg, trace=False)
    st = rep.status_code.cpu().numpy()
    assert np.array_equal(st, ref["status"])
    assert np.array_equal(rep.iterations.cpu().numpy(), ref["iters"])
    assert_res_parity({"res": rep.res.cpu().numpy()}, ref, tol=None)
    y, pi, lam, t = (v.cpu().numpy() for v in partial_expand_batch(rep, pmap, batch))
    lay2 = OcpLayout(ocb.dim)
    for i in range(n):
        short = dict(layout=lay2, y=ref["y"][i], pi=ref["pi"][i], lam=ref["lam"][i], t=ref["t"][i])
        ry, rpi, rlam, rt = co.partial_expand(qps[i], cq[i][1], short)
        for k, a, r in (("y", y[i], ry), ("pi", pi[i], rpi), ("lam", lam[i], rlam), ("t", t[i], rt)):
            assert rel_err(a, r) <= 1e-8, (i, k, rel_err(a, r))


def test_gpu_config4_partial_path_matches_reference_goldens(cuda, speed_arg, golden):
    """Full-size config 4 partial path on the GPU against the reference's own
    partial_condense -> solve -> partial_expand output (pcond_full.npz)."""
    from test_gpu_parity import assert_res_parity

    g = golden("pcond_full")
    idx = [int(i) for i in g["qps"]]
    batch = make_batch(4, batch=max(idx) + 1).select(idx)
    cb, pmap = partial_condense_batch(batch, 5)
    rep = solve_ocp_qp_batch(cb, speed_arg)
    st, its = rep.status_code.cpu().numpy(), rep.iterations.cpu().numpy()
    fl, res = rep.flops.cpu().numpy(), rep.res.cpu().numpy()
    full = [v.cpu().numpy() for v in partial_expand_batch(rep, pmap, batch)]
    for j, i in enumerate(idx):
        assert int(st[j]) == int(g[f"q{i}_short_status"])
        assert int(its[j]) == int(g[f"q{i}_short_iters"])
        assert int(fl[j]) == int(g[f"q{i}_short_flops"])
        assert_res_parity({"res": res[j:j + 1]}, {"res": g[f"q{i}_short_res"][None],
                                                   "status": st[j:j + 1]}, tol=1e-8)
        for k, v in zip(("y", "pi", "lam", "t"), full):
            assert rel_err(v[j], g[f"q{i}_full_{k}"]) <= 1e-8, (i, k)
