"""Multi-GPU plumbing for the sharded workloads (one process per GPU, torch.distributed).

Trajectories (and sweep points) are split into contiguous blocks [g*N/P, (g+1)*N/P). The only
exchange step is the ensemble mean: every rank all-gathers the per-block pairwise sums and the
completed-trajectory counts (NCCL over NVLink on GPUs; gloo in the CPU tests) and combines them in
the reference's pairwise bracket (trajectories.cpp:17-22, 82-83) with qsg_ensemble_combine.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int):
    """Contiguous block of rank `rank`: [n*rank//world, n*(rank+1)//world)."""
    return n * rank // world, n * (rank + 1) // world


def gather_block_sums(block_sum: np.ndarray, n_ok: int, world: int, device=None):
    """All-gather (block_sum, n_ok) from every rank; returns (list of sums, list of n_ok)."""
    import torch
    import torch.distributed as dist

    flat = np.concatenate([np.asarray(block_sum, np.complex128).reshape(-1), [complex(n_ok)]])
    t = torch.from_numpy(flat)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    sums, counts = [], []
    for p in parts:
        a = p.cpu().numpy()
        sums.append(a[:-1].reshape(np.asarray(block_sum).shape))
        counts.append(int(round(a[-1].real)))
    return sums, counts


def combine_mean(ntraj: int, world: int, sums, counts):
    """Deterministic ensemble mean of the gathered block sums (bitwise equal to one block when
    no trajectory failed)."""
    from . import ensemble_combine

    ranges = [shard_range(ntraj, k, world) for k in range(world)]
    return ensemble_combine(ranges, sums, int(sum(counts)))
