"""Diagnose the BIG team kernel on a random-structure case: traces of GPU (team), GPU (generic), oracle."""
import os, sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import qpgen, oracle as orc
import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch
from paper_2003_02547_b200 import solver as S
seed, N, nb, inf_side, mask_last = [(12, 7, 4, True, False), (17, 20, 200, True, True)][int(sys.argv[1]) if len(sys.argv) > 1 else 0]
dims, stages, dyn = qpgen.random_ocp_fields(seed, N=N, nx=60, nu=20, nb=nb, ng=0, ns=0, inf_side=inf_side,
                                            mask_last=mask_last, decay=0.9 / np.sqrt(60))
batch = OcpQpBatch.from_qps([qpgen.build_qp(pkg, dims, stages, dyn)])
arg = pkg.mode_preset("speed").with_tol(1e-6)
orc.build()
ref = orc.solve(batch, arg)
out = {}
for kind in ("auto", "generic"):
    os.environ.pop("OCPQP_GENERIC", None)
    if kind == "generic":
        os.environ["OCPQP_GENERIC"] = "1"
    S._PLANS.clear()
    rep = solve_ocp_qp_batch(batch, arg, trace=True)
    out[kind] = rep
    print(kind, S.get_plan(batch).info()["kernel"], "iters", int(rep.iterations[0]), "status", int(rep.status_code[0]))
print("oracle iters", ref["iters"], ref["status"])
tr_o = np.asarray(ref["trace"])[0]
np.set_printoptions(linewidth=200, precision=5)
for kind in ("auto", "generic"):
    tr = out[kind].trace.cpu().numpy()[0]
    print(kind)
    for i in range(max(int(out[kind].iterations[0]), int(ref["iters"][0])) + 1):
        print(i, tr[i] if i < len(tr) else None)
print("oracle")
for i in range(int(ref["iters"][0]) + 1):
    print(i, tr_o[i])
