"""User-built dense QPs (DenseQp + solve_dense_qp) vs the reference's
solve_dense_qp (tests/golden/dense.npz: random dense QPs with box, general,
soft rows and a masked side, speed 1e-8 and balance 1e-6).

The CPU test pins the oracle on the N = 0 form to the reference; the GPU test
runs the package's drop-in solve_dense_qp.  Bar: identical status and
iteration count; in speed mode identical counted flops and solutions within
1e-8; in balance mode solutions within 1e-6 (refinement-count flops may
differ, tests/modes_common.py).
"""

import numpy as np
import pytest

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, dense_to_ocp

from conftest import GOLDEN, rel_err


def _cases():
    src = (GOLDEN / "make_golden.py").read_text()
    ns = {}
    for key in ("DENSE_CASES = [", "DENSE_MODES = ("):
        start = src.index(key)
        end = src.index("\n\n", start)
        exec(src[start:end], {}, ns)
    gen_src = src[src.index("def dense_random_qp"):src.index("def dense():")]
    exec(gen_src, {"np": np}, ns)
    return ns["DENSE_CASES"], ns["DENSE_MODES"], ns["dense_random_qp"]


CASES, MODES, GEN = _cases()
PARAMS = [(c, m) for c in CASES for m in MODES]


def check(g, key, mode, status, iters, flops, y, lam, t):
    assert int(status) == int(g[f"{key}_status"])
    assert int(iters) == int(g[f"{key}_iters"])
    tol = 1e-8 if mode[1] == "speed" else 1e-6
    if mode[1] == "speed":
        assert int(flops) == int(g[f"{key}_flops"])
    for k, v in (("y", y), ("lam", lam), ("t", t)):
        assert rel_err(v, g[f"{key}_{k}"]) <= tol, k


@pytest.mark.parametrize("case,mode", PARAMS, ids=lambda p: str(p[0]) if isinstance(p, tuple) else p)
def test_oracle_dense_qp_matches_reference(golden, oracle, case, mode):
    g = golden("dense")
    q = GEN(pkg, *case)
    arg = pkg.mode_preset(mode[1]).with_tol(mode[2])
    ref = oracle.solve(OcpQpBatch.from_qps([dense_to_ocp(q)]), arg, nthreads=1)
    check(g, f"d{case[0]}_{mode[0]}", mode, ref["status"][0], ref["iters"][0], ref["flops"][0],
          ref["y"][0], ref["lam"][0], ref["t"][0])


@pytest.mark.gpu
@pytest.mark.parametrize("case,mode", PARAMS, ids=lambda p: str(p[0]) if isinstance(p, tuple) else p)
def test_gpu_solve_dense_qp_matches_reference(cuda, golden, case, mode):
    g = golden("dense")
    q = GEN(pkg, *case)
    rep = pkg.solve_dense_qp(q, pkg.mode_preset(mode[1]).with_tol(mode[2]))
    code = {"Success": 0, "MaxIter": 1, "MinStep": 2, "NaNDetected": 3, "Failure": 4}
    s = rep.solution
    check(g, f"d{case[0]}_{mode[0]}", mode, code[rep.status.value], rep.iterations,
          rep.stats.flops, s.y, s.lam, s.t)
    assert s.v.shape[0] == q.nv and s.sl_all.shape[0] == q.ns
