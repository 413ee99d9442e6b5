"""Multi-GPU sharding of the per-step compliance build.

One process per GPU.  The factor is replicated (each rank factorises its own
copy — it is needed by every rank's solves), the forward solve on the column
windows is replicated, and the expensive part — the Gram product U = Y^T Y —
is split by 64 x 64 output tiles, round-robin over ranks (tile pair index
t = A(A+1)/2 + B, owner t mod world).  Each rank writes only its tiles (and
their mirror) into a zero-filled U; one NCCL all-reduce (sum) assembles the
full U on every rank.  Every entry is produced by exactly one rank and the
others contribute exact zeros, so the result is bit-identical to the
single-GPU U.  The Newton loop then runs replicated (it is sequential and
HBM-bound; sharding W would cost an all-gather per iteration).
"""

from __future__ import annotations

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
    """Owner rank of every (sorted-order) entry (i, j) of an ncols x ncols U."""
    t = np.arange(ncols) // GRAM_TILE
    A = np.maximum(t[:, None], t[None, :])
    B = np.minimum(t[:, None], t[None, :])
    return (A * (A + 1) // 2 + B) % world


def reduce_shards(U, group=None) -> None:
    """Sum the per-rank partial U over the group (in place)."""
    import torch.distributed as dist

    dist.all_reduce(U, op=dist.ReduceOp.SUM, group=group)
