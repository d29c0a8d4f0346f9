"""Batch sharding across ranks (one process per GPU).

The path shards into independent QPs: rank r of W solves a
contiguous QP range with no data-path collective.  The only cross-rank
operations are the timing reduction (max over ranks) and an optional gather of
per-QP outcomes for reporting.
"""

from __future__ import annotations


def shard_range(B, rank, world):
    """Contiguous [lo, hi) QP range of ``rank`` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    lo = B * rank // world
    hi = B * (rank + 1) // world
    return lo, hi


def max_over_ranks(value, device=None):
    """Max of a scalar over all ranks (the contract's multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_outcomes(status, iterations, device=None):
    """All-gather per-rank (status, iterations) int tensors to every rank."""
    import torch
    import torch.distributed as dist

    s = torch.as_tensor(status, dtype=torch.int32, device=device)
    it = torch.as_tensor(iterations, dtype=torch.int32, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return s, it
    W = dist.get_world_size()
    n = torch.tensor([s.numel()], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(W)]
    dist.all_gather(sizes, n)
    m = int(max(int(x.item()) for x in sizes))
    pad = lambda x: torch.cat([x, torch.full((m - x.numel(),), -1, dtype=x.dtype, device=x.device)])
    gs = [torch.empty(m, dtype=torch.int32, device=device) for _ in range(W)]
    gi = [torch.empty(m, dtype=torch.int32, device=device) for _ in range(W)]
    dist.all_gather(gs, pad(s))
    dist.all_gather(gi, pad(it))
    out_s = torch.cat([g[: int(k.item())] for g, k in zip(gs, sizes)])
    out_i = torch.cat([g[: int(k.item())] for g, k in zip(gi, sizes)])
    return out_s, out_i
