"""Partial and full condensing of QPs with soft rows on the GPU vs the reference
(tests/golden/soft_cond.npz: condense / partial_condense outputs with their
slack data, the reference's solves of the condensed QPs and the expansions).

Slack data travels with its row (condensing.py:289-334, 523-534); expansion
routes the slacks and their multipliers back (:397-405, 592-601).  Same bar
as the hard-row condensing tests.
"""

import numpy as np
import pytest

from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200.condensing import (condense_batch, expand_batch,
                                              partial_condense_batch, partial_expand_batch)

from conftest import GOLDEN, rel_err
from test_condense_oracle import source_qp
from test_fcond_oracle import finite

pytestmark = pytest.mark.gpu

DMAP = {"H": "R", "g": "r", "lb": "lb", "ub": "ub", "C": "D", "lg": "lg", "ug": "ug",
        "maskl": "maskl", "masku": "masku", "Zl": "Zl", "Zu": "Zu", "zl": "zl", "zu": "zu",
        "sl_lb": "sl_lb", "su_lb": "su_lb"}
PFIELDS = ("Q", "S", "R", "q", "r", "lb", "ub", "C", "D", "lg", "ug", "maskl", "masku",
           "Zl", "Zu", "zl", "zu", "sl_lb", "su_lb")


def soft_cases():
    src = (GOLDEN / "make_golden.py").read_text()
    start = src.index("SOFT_CASES = [")
    end = src.index("]\n", start) + 1
    ns = {}
    exec(src[start:end], {"dict": dict, "True": True, "None": None}, ns)
    return ns["SOFT_CASES"]


@pytest.mark.parametrize("case", soft_cases(), ids=lambda c: c[0])
def test_gpu_full_condense_soft_rows(cuda, speed_arg, golden, case):
    name, src, keep, _ = case
    g = golden("soft_cond")
    batch = OcpQpBatch.from_qps([source_qp(src)])
    cb, cmap = condense_batch(batch, keep)
    nv, ne, nb, ng, ns, kept = (int(v) for v in g[f"{name}_dims"])
    assert (cmap.nv, int(cb.dim.nb[0]), int(cb.dim.ng[0]), int(cb.dim.ns[0])) == (nv, nb, ng, ns)
    q = cb.numpy().qp(0)
    assert np.array_equal(q.get_field("idxb", 0), g[f"{name}_idxb"])
    assert np.array_equal(q.get_field("idxs", 0), g[f"{name}_idxs"])
    for f, o in DMAP.items():
        assert rel_err(finite(q.get_field(o, 0)).reshape(-1),
                       finite(g[f"{name}_{f}"]).reshape(-1)) <= 1e-12, f
    rep = solve_ocp_qp_batch(cb, speed_arg)
    assert int(rep.status_code.cpu()[0]) == int(g[f"{name}_dense_status"])
    assert int(rep.iterations.cpu()[0]) == int(g[f"{name}_dense_iters"])
    assert int(rep.flops.cpu()[0]) == int(g[f"{name}_dense_flops"])
    for k in ("y", "lam", "t"):
        assert rel_err(getattr(rep, k).cpu().numpy()[0], g[f"{name}_dense_{k}"]) <= 1e-8, k
    y, pi, lam, t = expand_batch(rep, cmap, batch)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v.cpu().numpy()[0], g[f"{name}_full_{k}"]) <= 1e-8, k
    dense = tuple(g[f"{name}_dense_{k}"][None] for k in ("y", "pi", "lam", "t"))
    y, pi, lam, t = expand_batch(dense, cmap, batch)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v.cpu().numpy()[0], g[f"{name}_full_{k}"]) <= 1e-12, ("ref-dense", k)


@pytest.mark.parametrize("case", soft_cases(), ids=lambda c: c[0])
def test_gpu_partial_condense_soft_rows(cuda, speed_arg, golden, case):
    name, src, _, N1 = case
    g = golden("soft_cond")
    batch = OcpQpBatch.from_qps([source_qp(src)])
    cb, pmap = partial_condense_batch(batch, N1)
    dims = g[f"{name}_p_dims"]
    assert cb.dim.N == dims.shape[1] - 1
    assert list(cb.dim.ns) == list(dims[4]) and list(cb.dim.nu) == list(dims[1])
    q2 = cb.numpy().qp(0)
    for k in range(cb.dim.N + 1):
        assert np.array_equal(q2.get_field("idxb", k), g[f"{name}_p_s{k}_idxb"])
        assert np.array_equal(q2.get_field("idxs", k), g[f"{name}_p_s{k}_idxs"])
        for f in PFIELDS:
            assert rel_err(finite(q2.get_field(f, k)).reshape(-1),
                           finite(g[f"{name}_p_s{k}_{f}"]).reshape(-1)) <= 1e-12, (k, f)
        if k < cb.dim.N:
            for f in ("A", "B", "b"):
                assert rel_err(q2.get_field(f, k).reshape(-1),
                               g[f"{name}_p_s{k}_{f}"].reshape(-1)) <= 1e-12, (k, f)
    rep = solve_ocp_qp_batch(cb, speed_arg)
    assert int(rep.status_code.cpu()[0]) == int(g[f"{name}_short_status"])
    assert int(rep.iterations.cpu()[0]) == int(g[f"{name}_short_iters"])
    assert int(rep.flops.cpu()[0]) == int(g[f"{name}_short_flops"])
    y, pi, lam, t = partial_expand_batch(rep, pmap, batch)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v.cpu().numpy()[0], g[f"{name}_pfull_{k}"]) <= 1e-8, k
    short = tuple(g[f"{name}_short_{k}"][None] for k in ("y", "pi", "lam", "t"))
    y, pi, lam, t = partial_expand_batch(short, pmap, batch)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v.cpu().numpy()[0], g[f"{name}_pfull_{k}"]) <= 1e-12, ("ref-short", k)
