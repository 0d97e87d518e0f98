"""Multi-GPU plumbing for the sharded workloads (one process per GPU, torch.distributed).

Trajectories (and sweep points) are split into contiguous shards made of whole subtrees ("leaves")
of run_ensemble's pairwise bracket (trajectories.cpp:17-22): the bracket's nodes at depth
D = log2(P) for a power-of-two world and three levels deeper otherwise, assigned in order so every
rank gets about N/P trajectories. The only exchange step is the ensemble mean: every rank all-gathers
its per-leaf pairwise sums and completed-trajectory count (the product's NCCL communicator,
qsg_comm_allgather, over NVLink on GPUs; torch.distributed with gloo in the CPU tests) and all ranks
combine the leaves in the reference's bracket (qsg_ensemble_combine), bit for bit the single-device
mean when no trajectory failed. This restates qsim::ensemble_shards (csrc/host/evolve.cpp).
"""
from __future__ import annotations

import numpy as np


def ensemble_leaves(n: int, world: int):
    """Bracket subtrees [lo, hi) at depth D (split lo + (hi - lo)//2, trajectories.cpp:17-22)."""
    d = 0
    while (1 << d) < world:
        d += 1
    if (1 << d) != world:
        d += 3
    out = []

    def rec(lo, hi, k):
        if k == 0 or hi - lo <= 1:
            out.append((lo, hi))
            return
        mid = lo + (hi - lo) // 2
        rec(lo, mid, k - 1)
        rec(mid, hi, k - 1)

    rec(0, n, d)
    return out


def ensemble_shards(n: int, world: int):
    """[(begin, end, leaves)] per rank: contiguous runs of whole bracket subtrees, ~n/world each."""
    leaves = ensemble_leaves(n, world)
    shards, j = [], 0
    for k in range(world):
        target = n * (k + 1) // world
        mine = []
        while j < len(leaves) and (leaves[j][1] <= target or k == world - 1):
            mine.append(leaves[j])
            j += 1
        if not mine and j < len(leaves):
            mine.append(leaves[j])
            j += 1
        b = mine[0][0] if mine else n
        e = mine[-1][1] if mine else b
        shards.append((b, e, mine))
    return shards


def shard_range(n: int, rank: int, world: int):
    """Contiguous trajectory (or point) range of rank `rank`: whole bracket subtrees, ~n/world."""
    b, e, _ = ensemble_shards(n, world)[rank]
    return b, e


class ProductComm:
    """The product's NCCL communicator for one rank (qsg_comm_init_rank); rank 0 creates the id and
    torch.distributed broadcasts it (the bootstrap only)."""

    def __init__(self, ctx, rank: int, world: int):
        import ctypes as C

        import torch.distributed as dist

        from . import _check, lib

        L = lib()
        L.qsg_comm_unique_id.argtypes = [C.c_void_p]
        L.qsg_comm_init_rank.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]
        L.qsg_comm_allgather.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.qsg_comm_destroy.argtypes = [C.c_void_p]
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(L.qsg_comm_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        self._h = C.c_void_p()
        _check(L.qsg_comm_init_rank(ctx._h, world, rank, uid, C.byref(self._h)))
        self.world = world
        self._lib = L

    def allgather(self, a: np.ndarray) -> np.ndarray:
        from . import _check

        a = np.ascontiguousarray(a, np.float64).reshape(-1)
        out = np.empty(a.size * self.world)
        _check(self._lib.qsg_comm_allgather(self._h, a.ctypes.data, a.size, out.ctypes.data))
        return out.reshape(self.world, a.size)

    def close(self):
        if self._h:
            self._lib.qsg_comm_destroy(self._h)
            self._h = None


def gather_leaf_sums(leaf_sums, n_ok: int, n_leaves_max: int, world: int, comm=None, device=None):
    """All-gather every rank's (n_ok, leaf sums); returns (list per rank of leaf-sum lists, counts).
    comm: a ProductComm (NCCL inside the product); None = torch.distributed.all_gather."""
    shape = np.asarray(leaf_sums[0]).shape
    nv = int(np.prod(shape))
    flat = np.zeros(2 + 2 * nv * n_leaves_max)
    flat[0], flat[1] = n_ok, len(leaf_sums)
    for k, s in enumerate(leaf_sums):
        flat[2 + 2 * nv * k:2 + 2 * nv * (k + 1)] = np.asarray(s, np.complex128).reshape(-1).view(np.float64)
    if comm is not None:
        parts = comm.allgather(flat)
    else:
        import torch
        import torch.distributed as dist

        t = torch.from_numpy(flat)
        if device is not None:
            t = t.to(device)
        ps = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(ps, t)
        parts = np.stack([p.cpu().numpy() for p in ps])
    sums, counts = [], []
    for p in parts:
        counts.append(int(round(p[0])))
        nl = int(round(p[1]))
        sums.append([p[2 + 2 * nv * k:2 + 2 * nv * (k + 1)].view(np.complex128).reshape(shape) for k in range(nl)])
    return sums, counts


def combine_leaves(n: int, world: int, sums, counts):
    """Deterministic ensemble mean from every rank's gathered leaf sums (bitwise equal to one
    block when no trajectory failed)."""
    from . import ensemble_combine

    ranges, flat = [], []
    for (b, e, leaves), s in zip(ensemble_shards(n, world), sums):
        ranges.extend(leaves)
        flat.extend(s)
    return ensemble_combine(ranges, flat, int(sum(counts)))


# ---- one block per rank (power-of-two worlds), kept for the sweep and older callers ------------
def gather_block_sums(block_sum: np.ndarray, n_ok: int, world: int, device=None, comm=None):
    """All-gather (block_sum, n_ok) from every rank; returns (list of sums, list of n_ok)."""
    s, c = gather_leaf_sums([block_sum], n_ok, 1, world, comm=comm, device=device)
    return [x[0] for x in s], c


def combine_mean(ntraj: int, world: int, sums, counts):
    """Mean from one block sum per rank (the rank's whole shard)."""
    from . import ensemble_combine

    ranges = [shard_range(ntraj, k, world) for k in range(world)]
    return ensemble_combine(ranges, sums, int(sum(counts)))
