"""CPU tests of the multi-rank host logic with torch.distributed gloo, world size 2.

The sharded mcsolve path (bench.py secondary) splits trajectories into contiguous
blocks, all-gathers per-block pairwise sums and combines them in the reference bracket. Here the
per-trajectory data is synthetic; the combine must equal the single-process pairwise mean
(trajectories.cpp:17-22,82-83) bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_21440_b200.dist import (combine_leaves, combine_mean, ensemble_shards, gather_block_sums,
                                        gather_leaf_sums, shard_range)

NTRAJ, NE, NT = 10000, 1, 100


def pairwise(mats, lo, hi):
    if hi - lo == 1:
        return mats[lo].copy()
    mid = lo + (hi - lo) // 2
    return pairwise(mats, lo, mid) + pairwise(mats, mid, hi)


def cdiv(z, n):
    """Complex(N, 0) division as libgcc's __divdc3 does it for a real divisor (componentwise);
    numpy's complex division rounds differently."""
    return z.real / n + 1j * (z.imag / n)


def synthetic():
    rng = np.random.default_rng(7)
    return rng.standard_normal((NTRAJ, NE, NT)) + 1j * rng.standard_normal((NTRAJ, NE, NT))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    data = synthetic()
    shards = ensemble_shards(NTRAJ, world)
    b, e, leaves = shards[rank]
    # per-leaf pairwise sums, as qsg_mcsolve's range_sums return them
    ls = [pairwise(list(data[lo:hi]), 0, hi - lo) for lo, hi in leaves]
    sums, counts = gather_leaf_sums(ls, e - b, max(len(s[2]) for s in shards), world)
    mean = combine_leaves(NTRAJ, world, sums, counts)
    q.put((rank, mean, counts))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_combine_bitwise_equals_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = synthetic()
    ref = cdiv(pairwise(list(data), 0, NTRAJ), NTRAJ)
    for rank, mean, counts in out:
        assert sum(counts) == NTRAJ and max(counts) - min(counts) <= NTRAJ // (8 * world) + 1
        assert np.array_equal(mean.view(np.float64), ref.view(np.float64)), rank


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_blocks_align_with_pairwise_bracket(world):
    """10,000 trajectories in P in {1,2,4,8} contiguous blocks sit on the top levels of the
    pairwise_sum split, so the block-combine is exact (no mid-block split)."""
    data = synthetic()[:, :, :4]
    sums, counts = [], []
    for r in range(world):
        b, e = shard_range(NTRAJ, r, world)
        sums.append(pairwise(list(data[b:e]), 0, e - b))
        counts.append(e - b)
    mean = combine_mean(NTRAJ, world, sums, counts)
    ref = cdiv(pairwise(list(data), 0, NTRAJ), NTRAJ)
    assert np.array_equal(mean.view(np.float64), ref.view(np.float64))


def test_misaligned_blocks_rejected():
    import paper_2504_21440_b200 as q
    with pytest.raises(q.QsgError):
        q.ensemble_combine([(0, 3), (3, 10)], [np.ones((1, 2)), np.ones((1, 2))], 10)


@pytest.mark.parametrize("world", [1, 2, 3, 5, 6, 7, 8])
def test_ensemble_shards_tile_and_balance(world):
    """Shards are contiguous, tile [0, N), are made of whole bracket subtrees, and stay balanced
    for any world size (non-power-of-two worlds)."""
    shards = ensemble_shards(NTRAJ, world)
    assert shards[0][0] == 0 and shards[-1][1] == NTRAJ
    for (b0, e0, _), (b1, e1, _) in zip(shards, shards[1:]):
        assert e0 == b1
    sizes = [e - b for b, e, _ in shards]
    assert max(sizes) - min(sizes) <= NTRAJ // (8 * world) + 2
    data = synthetic()[:, :, :3]
    sums = [[pairwise(list(data[lo:hi]), 0, hi - lo) for lo, hi in lv] for _, _, lv in shards]
    mean = combine_leaves(NTRAJ, world, sums, sizes)
    ref = cdiv(pairwise(list(data), 0, NTRAJ), NTRAJ)
    assert np.array_equal(mean.view(np.float64), ref.view(np.float64))
