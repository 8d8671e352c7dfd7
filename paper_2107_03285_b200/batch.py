"""Instance partitioning and the end-of-run gather for batched SGN (BASELINE config 5).

Independent design instances shard with no data-path collective: rank r of W owns a
contiguous instance range; every rank runs its instances as one device batch; a single
all-gather at the end collects per-instance results (dp, objective trajectory, status) on
every rank (NCCL over NVLink on the GPU box, gloo in the CPU tests).  No reduction is
involved, so gathered results are bitwise independent of W.
"""
from __future__ import annotations

import numpy as np


def partition(n_total: int, world: int, rank: int) -> range:
    """Contiguous, balanced instance range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(int(n_total), int(world))
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_instances(local: np.ndarray, n_total: int, world: int, rank: int, device=None) -> np.ndarray:
    """All-gather per-instance rows (local: [n_local, m]) into [n_total, m] on every rank."""
    import torch
    import torch.distributed as dist
    local = np.ascontiguousarray(local, dtype=np.float64)
    m = local.shape[1] if local.ndim == 2 else 1
    local = local.reshape(-1, m)
    cap = max(len(partition(n_total, world, r)) for r in range(world))
    buf = np.zeros((cap, m))
    buf[:local.shape[0]] = local
    t = torch.as_tensor(buf, device=device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    rows = []
    for r in range(world):
        k = len(partition(n_total, world, r))
        rows.append(outs[r].cpu().numpy()[:k])
    return np.concatenate(rows, axis=0)
