import sys, torch, numpy as np
sys.path.insert(0,'/root/repo')
from paper_2003_02547_b200 import mode_preset, solve_ocp_qp_batch
from paper_2003_02547_b200.generators import make_batch
from paper_2003_02547_b200.solver import get_plan
arg = mode_preset("speed").with_tol(1e-8)
dev = make_batch(4).to("cuda")
def run(n=4):
    ts=[]
    for _ in range(n):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); rep=solve_ocp_qp_batch(dev,arg,trace=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts, rep
t0, r0 = run()
get_plan(dev).dispatch_hint(True)
t1, r1 = run(6)
print("no hint", [round(x,2) for x in t0]); print("hint", [round(x,2) for x in t1])
for k in ("y","pi","lam","t"):
    print(k, float((getattr(r0,k)-getattr(r1,k)).abs().max()))
print("iters equal", bool((r0.iterations==r1.iterations).all()), "status", bool((r0.status_code==r1.status_code).all()))
get_plan(dev).dispatch_hint(False)
t2,_=run(3); print("off again", [round(x,2) for x in t2])
