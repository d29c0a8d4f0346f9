import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, qpgen
import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200 import OcpQpBatch, solve_ocp_qp_batch, mode_preset
from paper_2003_02547_b200 import solver as S
from oracle import oracle as O
from conftest import rel_err
arg = mode_preset("speed").with_tol(1e-8)
for (nx,nu,ng,seed,N,nb,i,m) in [(24,4,0,13,12,2,False,True),(8,3,0,13,12,2,False,True),(24,4,0,12,7,4,True,False)]:
    d,s,dy = qpgen.random_ocp_fields(seed,N=N,nx=nx,nu=nu,nb=nb,ng=ng,ns=0,inf_side=i,mask_last=m)
    b = OcpQpBatch.from_qps([qpgen.build_qp(pkg,d,s,dy)])
    ref = O.solve(b, arg)
    out = {}
    for kind, env in [("team", {}), ("generic", {"OCPQP_GENERIC": "1"})]:
        os.environ.pop("OCPQP_GENERIC", None); os.environ.update(env); S._PLANS.clear()
        r = solve_ocp_qp_batch(b, arg)
        out[kind] = r
        print(nx,nu,seed,kind, S.get_plan(b).info()["kernel"], int(r.iterations[0]), int(ref["iters"][0]),
              {k: rel_err(getattr(r,k).cpu().numpy()[0], ref[k][0]) for k in ("y","pi","lam","t")})
    print("  team vs generic y:", rel_err(out["team"].y.cpu().numpy()[0], out["generic"].y.cpu().numpy()[0]),
          " |y|max", np.abs(ref["y"]).max(), " lam max", np.abs(ref["lam"]).max(), "res", ref["res"][0])
