"""Multi-process (gloo, world_size 2 and 3, CPU) checks of the N>1 host logic.

parallel.run_split drives the column-split compliance protocol (plan, forward
of the rank's columns, all-gather of the compact Y, Gram tiles t -> rank
t mod world, all-gather of the tile buffers, scatter).  Here it runs over real
gloo collectives with a numpy model of the kernels (per-column triangular
solves, 64 x 64 Gram tiles), and every rank must end with exactly the
single-process C = Y^T Y.  The same orchestration calls the CUDA kernels on
the GPU (tests/test_gpu_parallel.py checks those against one GPU bit for bit).
"""

import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_06946_b200.parallel import GRAM_TILE, all_gather, run_split, tile_owner


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


class NumpySteps:
    """The kernels' contract in numpy: Y = L^-1 E column by column, Gram tiles."""

    def __init__(self, L, E, rank, world):
        self.L, self.E, self.rank, self.world = L, E, rank, world
        self.n, self.k = E.shape
        b = np.linspace(0, self.k, world + 1).astype(int)
        self.cols = [(b[q], b[q + 1]) for q in range(world)]
        nt = (self.k + GRAM_TILE - 1) // GRAM_TILE
        self.npairs = nt * (nt + 1) // 2
        self.per_rank = (self.npairs + world - 1) // world
        self.C = None

    def plan(self):
        send = max(b - a for a, b in self.cols) * self.n
        return max(send, 1), self.per_rank * GRAM_TILE * GRAM_TILE, (0.0, 0.0)

    def forward(self, ysend):
        a, b = self.cols[self.rank]
        ysend.zero_()
        for j in range(a, b):
            y = sla.solve_triangular(self.L, self.E[:, j], lower=True)
            ysend[(j - a) * self.n:(j - a + 1) * self.n] = torch.from_numpy(y)

    def _Y(self, yall):
        send = yall.numel() // self.world
        Y = np.zeros((self.n, self.k))
        for q, (a, b) in enumerate(self.cols):
            blk = yall[q * send:q * send + (b - a) * self.n].numpy().reshape(b - a, self.n)
            Y[:, a:b] = blk.T
        return Y

    @staticmethod
    def _tile(t):
        A = int((np.sqrt(8 * t + 1) - 1) // 2)
        while (A + 1) * (A + 2) // 2 <= t:
            A += 1
        while A * (A + 1) // 2 > t:
            A -= 1
        return A, t - A * (A + 1) // 2

    def gram(self, yall, tiles):
        Y = np.zeros((self.n, self.npairs and ((self.k + GRAM_TILE - 1) // GRAM_TILE) * GRAM_TILE))
        Y[:, :self.k] = self._Y(yall)
        tiles.zero_()
        for slot, t in enumerate(range(self.rank, self.npairs, self.world)):
            A, B = self._tile(t)
            blk = Y[:, A * GRAM_TILE:(A + 1) * GRAM_TILE].T @ Y[:, B * GRAM_TILE:(B + 1) * GRAM_TILE]
            tiles[slot * GRAM_TILE ** 2:(slot + 1) * GRAM_TILE ** 2] = torch.from_numpy(blk.ravel())

    def finish(self, tiles_all):
        kp = ((self.k + GRAM_TILE - 1) // GRAM_TILE) * GRAM_TILE
        C = np.zeros((kp, kp))
        T = tiles_all.numpy()
        for t in range(self.npairs):
            A, B = self._tile(t)
            off = ((t % self.world) * self.per_rank + t // self.world) * GRAM_TILE ** 2
            blk = T[off:off + GRAM_TILE ** 2].reshape(GRAM_TILE, GRAM_TILE)
            C[A * GRAM_TILE:(A + 1) * GRAM_TILE, B * GRAM_TILE:(B + 1) * GRAM_TILE] = blk
            C[B * GRAM_TILE:(B + 1) * GRAM_TILE, A * GRAM_TILE:(A + 1) * GRAM_TILE] = blk.T
        self.C = C[:self.k, :self.k]


def _problem():
    rng = np.random.default_rng(0)
    n, k = 90, 150
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    L = np.linalg.cholesky(A)
    E = np.zeros((n, k))
    E[rng.integers(0, n, k), np.arange(k)] = 1.0
    return L, E


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, E = _problem()
    steps = NumpySteps(L, E, rank, world)

    # the production gather (parallel.all_gather: all_gather_into_tensor), over gloo
    run_split(steps, world, all_gather(), lambda n: torch.empty(int(n), dtype=torch.float64))
    out[rank] = steps.C
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_split_protocol_reproduces_one_process(world):
    L, E = _problem()
    single = NumpySteps(L, E, 0, 1)
    run_split(single, 1, lambda o, i: o.copy_(i), lambda n: torch.empty(int(n), dtype=torch.float64))
    Y = sla.solve_triangular(L, E, lower=True)
    assert np.abs(single.C - Y.T @ Y).max() <= 1e-12 * np.abs(single.C).max()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(out[r], single.C)


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
