"""Multi-rank path on CPU: world_size-2 gloo ranks shard the batch (replicas).

bench.py --gpus N runs one process per GPU; each solves a contiguous QP shard
with no data-path collective, the step time is the max over ranks and outcomes
can be gathered.  Here the per-rank solver is the CPU oracle (no GPU in this
container), so the test covers the sharding / reduction / gather logic.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle"), str(root / "tests")]
    import torch.distributed as dist

    import oracle as orc
    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.sharding import gather_outcomes, max_over_ranks, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(B, rank, world)
    batch = make_batch(1, batch=B).select(range(lo, hi))
    out = orc.solve(batch, mode_preset("speed").with_tol(1e-8), nthreads=1, trace=False)
    tmax = max_over_ranks(float(rank + 1))
    s, it = gather_outcomes(out["status"], out["iters"])
    if rank == 0:
        q.put((tmax, s.numpy().tolist(), it.numpy().tolist()))
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_solve(oracle):
    B = 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, status, iters = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    from paper_2003_02547_b200 import mode_preset
    from paper_2003_02547_b200.generators import make_batch

    ref = oracle.solve(make_batch(1, batch=B), mode_preset("speed").with_tol(1e-8), trace=False)
    assert status == ref["status"].tolist()
    assert iters == ref["iters"].tolist()
