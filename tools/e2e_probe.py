"""Break down the host-buffer (e2e) path of config 1: H2D alone, the solve
alone, and the whole ocpqp_solve_host call, CUDA-event timed."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.solver import solve_ocp_qp_batch, solve_ocp_qp_host

    arg = mode_preset("speed").with_tol(1e-8)
    b = make_batch(1)
    hb = b.pin_memory()
    dev = b.to("cuda")
    B, lay = b.B, b.layout
    out = dict(y=torch.empty((B, lay.ny), dtype=torch.float64).pin_memory(),
               pi=torch.empty((B, lay.ne), dtype=torch.float64).pin_memory(),
               lam=torch.empty((B, lay.nc), dtype=torch.float64).pin_memory(),
               t=torch.empty((B, lay.nc), dtype=torch.float64).pin_memory(),
               status=torch.empty(B, dtype=torch.int32).pin_memory(),
               iters=torch.empty(B, dtype=torch.int32).pin_memory(),
               res=torch.empty((B, 5), dtype=torch.float64).pin_memory(),
               flops=torch.empty(B, dtype=torch.int64).pin_memory(), trace=None)
    s = torch.cuda.current_stream()

    def ev(fn, n=20):
        ts = []
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)), float(np.min(ts))

    for _ in range(5):
        solve_ocp_qp_host(hb, arg, out=out, stream=s)
        solve_ocp_qp_batch(dev, arg)
    hbytes = sum(int(v.numel()) * 8 for v in hb.fields.values())
    src = torch.empty(hbytes // 8, dtype=torch.float64).pin_memory()
    dst = torch.empty(hbytes // 8, dtype=torch.float64, device="cuda")
    print("h2d %d B" % hbytes, ev(lambda: dst.copy_(src, non_blocking=True)))
    print("device solve", ev(lambda: solve_ocp_qp_batch(dev, arg)))
    print("host solve (e2e)", ev(lambda: solve_ocp_qp_host(hb, arg, out=out, stream=s)))
    t0 = time.perf_counter()
    for _ in range(20):
        solve_ocp_qp_host(hb, arg, out=out, stream=s)
    print("host solve wall ms", (time.perf_counter() - t0) / 20 * 1e3)


if __name__ == "__main__":
    main()
