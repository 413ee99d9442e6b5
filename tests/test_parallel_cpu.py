"""Multi-process (gloo, world_size 2, CPU) checks of the N>1 host logic: the Gram
tile ownership partitions U exactly once, and the zero-filled per-rank shards
summed by all-reduce reproduce the single-process U bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_06946_b200.parallel import tile_owner


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tile_ownership_partitions_every_entry_once():
    for ncols in (1, 63, 64, 65, 300, 1500):
        for world in (1, 2, 3, 8):
            own = tile_owner(ncols, world)
            assert own.shape == (ncols, ncols)
            assert np.array_equal(own, own.T)  # a tile and its mirror share the owner
            counts = np.bincount(own.ravel(), minlength=world)
            assert counts.sum() == ncols * ncols
            if ncols >= 300 and world > 1:  # round robin keeps the load balanced
                assert counts.max() <= 1.35 * counts.mean()


def _worker(rank, world, port, U_full, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    own = tile_owner(U_full.shape[0], world)
    shard = torch.as_tensor(np.where(own == rank, U_full, 0.0))
    dist.all_reduce(shard, op=dist.ReduceOp.SUM)
    out[rank] = shard.numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_shard_reduce_is_exact():
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((40, 150))
    U = Y.T @ Y
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, U, out), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(out[r], U)


def test_cfg4_copy_partition_covers_every_copy_once():
    """Scene-parallel cfg4: ranks take contiguous, disjoint copy ranges that cover
    all copies for every world size the scaling run uses (bench.cfg4_copy_range)."""
    import bench

    for world in (1, 2, 3, 4, 8):
        seen = []
        for rank in range(world):
            a, b = bench.cfg4_copy_range(rank, world)
            assert 0 <= a <= b <= bench.CFG4_COPIES
            seen.extend(range(a, b))
        assert seen == list(range(bench.CFG4_COPIES))


def test_cfg4_draws_are_per_copy_seeded():
    """Copy i's tilt, mu and jitter depend only on i (rng([4, i])), so any rank
    split reproduces the same copies."""
    from paper_2306_06946_b200.batch import cfg4_draws

    t_all, m_all, j_all = cfg4_draws(0, 6, 12)
    t_part, m_part, j_part = cfg4_draws(3, 3, 12)
    assert np.array_equal(t_all[3:], t_part) and np.array_equal(m_all[3:], m_part)
    assert np.array_equal(j_all[3:], j_part)
    assert (t_all >= 0).all() and (t_all <= 20).all() and (m_all >= 0.2).all() and (m_all <= 0.8).all()
