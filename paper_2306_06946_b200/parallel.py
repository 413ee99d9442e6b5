"""Multi-GPU sharding of the per-step compliance build.

One process per GPU, NCCL through torch.distributed.  The per-step W_g build
(reference assemble_Wg constraints.py:155-179 -> solve_multi linalg.py:98-106)
is split by right-hand-side COLUMNS with the factor replicated (every rank
factorises its own copy; it needs it for its solves):

1. plan     every rank sorts the columns of E (the touched DoFs) by their first
            supernode and takes a contiguous range of them, balanced by
            forward-solve work (``cnb_chol_compliance_plan``);
2. forward  rank r forward-solves only its columns, Y_r = L^-1 P E_r, into a
            compact buffer (``cnb_chol_compliance_forward``);
3. gather   ``all_gather_into_tensor`` of the compact Y_r (NCCL over NVLink);
4. gram     every rank unpacks the full Y and computes the 64 x 64 Gram tiles of
            C = Y^T Y it owns (tile t -> rank t mod world) into a tile buffer
            (``cnb_chol_compliance_gram``);
5. gather   ``all_gather_into_tensor`` of the tile buffers;
6. finish   every rank scatters every tile into C (``cnb_chol_compliance_finish``).

Each column's forward solve and each tile's Gram sum are computed exactly as on
one GPU, so C is bit-identical for every world size.  The Newton loop then runs
replicated on every rank (it is sequential and HBM-bound; sharding W would
cost an all-gather per iteration).  Batched independent scenes (cfg4) are
split per rank with no collective (bench.py cfg4_copy_range).

``run_split`` is written against an abstract step object and gather function
so the same orchestration runs over gloo on CPU in the tests
(tests/test_parallel_cpu.py) and over NCCL with the CUDA kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

GRAM_TILE = 64


def world_info(group=None) -> tuple[int, int]:
    """(rank, world) of the given / default process group, (0, 1) without one."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(group), dist.get_world_size(group)
    except Exception:
        pass
    return 0, 1


def tile_owner(ncols: int, world: int) -> np.ndarray:
    """Owner rank of every (sorted-order) entry (i, j) of an ncols x ncols C."""
    t = np.arange(ncols) // GRAM_TILE
    A = np.maximum(t[:, None], t[None, :])
    B = np.minimum(t[:, None], t[None, :])
    return (A * (A + 1) // 2 + B) % world


def all_gather(group=None):
    """gather(out, inp): rank-major concatenation of every rank's ``inp`` into ``out``."""
    import torch.distributed as dist

    def gather(out, inp):
        dist.all_gather_into_tensor(out, inp, group=group)

    return gather


def run_split(steps, world: int, gather, alloc) -> dict:
    """The split protocol: plan, forward, gather Y, gram, gather tiles, finish.

    ``steps`` provides plan() -> (send_count, tile_count, flops), forward(ysend),
    gram(yall, tiles), finish(tiles_all); ``alloc(n)`` returns an n-element
    buffer on the collective's device."""
    send, ntile, flops = steps.plan()
    ysend = alloc(send)
    yall = alloc(world * send)
    steps.forward(ysend)
    gather(yall, ysend)
    tiles = alloc(ntile)
    tiles_all = alloc(world * ntile)
    steps.gram(yall, tiles)
    gather(tiles_all, tiles)
    steps.finish(tiles_all)
    return {"send_doubles": send, "tile_doubles": ntile, "flops": flops}


class KernelSteps:
    """run_split steps backed by the library (one factor handle, one object)."""

    def __init__(self, F, ncols, colptr, rowidx, vals, out, ldu, rank, world):
        self.F, self.ncols = F, ncols
        self.colptr, self.rowidx, self.vals = colptr, rowidx, vals
        self.out, self.ldu, self.rank, self.world = out, ldu, rank, world

    def plan(self):
        from . import _lib

        sizes = (ctypes.c_int64 * 4)()
        fl = (ctypes.c_double * 2)()
        _lib.call("cnb_chol_compliance_plan", self.F._h, self.ncols, self.colptr.ctypes.data, self.rowidx.ctypes.data,
                  self.vals.ctypes.data, self.rank, self.world, sizes, fl, _lib.stream())
        self.columns = (int(sizes[2]), int(sizes[3]))
        return int(sizes[0]), int(sizes[1]), (float(fl[0]), float(fl[1]))

    def forward(self, ysend):
        from . import _lib

        _lib.call("cnb_chol_compliance_forward", self.F._h, ysend.data_ptr(), _lib.stream())

    def gram(self, yall, tiles):
        from . import _lib

        _lib.call("cnb_chol_compliance_gram", self.F._h, yall.data_ptr(), tiles.data_ptr(), _lib.stream())

    def finish(self, tiles_all):
        from . import _lib

        _lib.call("cnb_chol_compliance_finish", self.F._h, tiles_all.data_ptr(), self.out.data_ptr(), self.ldu,
                  _lib.stream())


def split_compliance(F, ncols, colptr, rowidx, vals, out, ldu, group=None, rank=None, world=None,
                     gather=None) -> dict:
    """C = E^T A^-1 E (or U = S A^-1 S^T) into ``out`` with the columns split over
    the process group (NCCL all-gathers); returns this rank's flops and sizes."""
    from . import _device as dv

    if rank is None or world is None:
        rank, world = world_info(group)
    steps = KernelSteps(F, ncols, colptr, rowidx, vals, out, ldu, rank, world)
    info = run_split(steps, world, gather or all_gather(group), lambda n: dv.empty(int(n)))
    info["columns"] = steps.columns
    return info
