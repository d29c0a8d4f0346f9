"""Pin the partial-condensing oracle (oracle/condense_oracle.py) to the reference.

tests/golden/pcond.npz holds the reference's partial_condense output fields,
its speed-mode solve of the condensed QP and the partial_expand result.
"""

import numpy as np
import pytest

import condense_oracle as co
import qpgen

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200.generators import make_batch
from paper_2003_02547_b200.layout import OcpLayout

from conftest import GOLDEN, rel_err


def pcond_cases():
    src = (GOLDEN / "make_golden.py").read_text()
    start = src.index("PCOND_CASES = [")
    end = src.index("]\n", src.index('("c1", ("cfg", 1, None), 5),')) + 1
    ns = {}
    exec(src[start:end], {"dict": dict}, ns)
    return ns["PCOND_CASES"]


def source_qp(src):
    if src[0] == "cfg":
        _, cfg, N = src
        return make_batch(cfg, batch=1, start=0, N=N).qp(0)
    seed, kw = src
    return qpgen.build_qp(pkg, *qpgen.random_ocp_fields(seed, **kw))


FIELDS = ("Q", "S", "R", "q", "r", "lb", "ub", "C", "D", "lg", "ug", "maskl", "masku")


@pytest.mark.parametrize("case", pcond_cases(), ids=lambda c: c[0])
def test_condense_oracle_matches_reference(golden, case):
    name, src, N1 = case
    g = golden("pcond")
    qp = source_qp(src)
    stages, blocks = co.partial_condense(qp, N1)
    assert len(stages) == len(blocks) == g[f"{name}_dims"].shape[1] - 1
    for k, st in enumerate(stages):
        assert np.array_equal(st["idxb"], g[f"{name}_s{k}_idxb"])
        for f in FIELDS + ("A", "B", "b"):
            ref = g[f"{name}_s{k}_{f}"]
            assert st[f].shape == ref.shape, (k, f)
            assert rel_err(np.nan_to_num(st[f], posinf=1e300, neginf=-1e300),
                           np.nan_to_num(ref, posinf=1e300, neginf=-1e300)) <= 1e-12, (k, f)


@pytest.mark.parametrize("case", pcond_cases(), ids=lambda c: c[0])
def test_expand_oracle_matches_reference(golden, case):
    name, src, N1 = case
    g = golden("pcond")
    qp = source_qp(src)
    _, blocks = co.partial_condense(qp, N1)
    dims = g[f"{name}_dims"]
    N2 = dims.shape[1] - 1
    sdim = pkg.OcpQpDim(N2, dims[0], dims[1], dims[2], dims[3])
    short = {k: g[f"{name}_short_{k}"] for k in ("y", "pi", "lam", "t")}
    short["layout"] = OcpLayout(sdim)
    y, pi, lam, t = co.partial_expand(qp, blocks, short)
    for k, v in (("y", y), ("pi", pi), ("lam", lam), ("t", t)):
        assert rel_err(v, g[f"{name}_full_{k}"]) <= 1e-11, k


def test_partial_path_oracle_config4_full_size(golden, oracle, speed_arg):
    """The oracle's partial path at BASELINE config 4's full size (N = 100 ->
    N2 = 20, nx = 60, nu = 20) against the reference's (pcond_full.npz):
    condensed-solve status, iterations, flops and final norms; expanded
    y / pi / lam / t within 1e-9 relative."""
    g = golden("pcond_full")
    qps_idx = [int(i) for i in g["qps"]]
    src = [make_batch(4, batch=1, start=i).qp(0) for i in qps_idx]
    cq = [co.partial_condensed_qp(q, 5) for q in src]
    cb = pkg.OcpQpBatch.from_qps([c[0] for c in cq])
    assert cb.dim.N == 20 and int(cb.dim.nu[0]) == 100 and int(cb.dim.ng[0]) == 240
    ref = oracle.solve(cb, speed_arg, nthreads=len(src), trace=False)
    lay2 = OcpLayout(cb.dim)
    for j, i in enumerate(qps_idx):
        assert int(ref["status"][j]) == int(g[f"q{i}_short_status"])
        assert int(ref["iters"][j]) == int(g[f"q{i}_short_iters"])
        assert int(ref["flops"][j]) == int(g[f"q{i}_short_flops"])
        r = g[f"q{i}_short_res"]
        assert np.all(np.abs(ref["res"][j] - r) <= 1e-8 * np.maximum(1.0, np.abs(r)))
        short = dict(layout=lay2, y=ref["y"][j], pi=ref["pi"][j], lam=ref["lam"][j], t=ref["t"][j])
        full = co.partial_expand(src[j], cq[j][1], short)
        for k, v in zip(("y", "pi", "lam", "t"), full):
            assert rel_err(v, g[f"q{i}_full_{k}"]) <= 1e-9, (i, k, rel_err(v, g[f"q{i}_full_{k}"]))
