"""Per-object mapping compliance U_o = S_o A_o^-1 S_o^T on the GPU factor.

Replaces the multi-RHS solve + sparse product of assemble_Wg
(/root/reference/pkg/src/contactnewton/constraints.py:175-178): instead of
X = A^-1 S^T (n x 3p dense) and S X, the library forward-solves only the
elimination paths of S^T's columns (Y = L^-1 P S^T) and forms U = Y^T Y with
fp64 tensor-core tiles (csrc/chol.cu: fwd_kernel sparse mode, gram_kernel).
Only the rows/columns of the pairs the object takes part in are formed.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as dv
from . import _lib


def object_compliance(S, F, dim: int, stats: dict | None = None, group=None, shard: bool = True):
    """U_o for one object.  Under torch.distributed (world > 1) the Gram tiles are
    split across ranks and summed with one all-reduce (parallel.py)."""
    from .constraints import ObjectCompliance
    from .parallel import reduce_shards, world_info

    rank, world = world_info(group) if shard else (0, 1)

    idx, side = S.idx, S.side
    mo = len(idx)
    d = dv.device()
    full = mo == dim // 3 and (mo == 0 or np.array_equal(idx, np.arange(mo)))
    U = dv.empty((3 * mo, 3 * mo))
    if mo:
        rows = (3 * idx[:, None] + np.arange(3)).ravel()
        csr = S.csr
        colptr = np.zeros(3 * mo + 1, dtype=np.int64)
        counts = np.diff(csr.indptr)[rows]
        colptr[1:] = np.cumsum(counts)
        starts = csr.indptr[rows]
        sel = np.concatenate([np.arange(s, s + c) for s, c in zip(starts, counts)]) if counts.sum() else \
            np.zeros(0, dtype=np.int64)
        rowidx = np.ascontiguousarray(csr.indices[sel], dtype=np.int64)
        vals = np.ascontiguousarray(csr.data[sel], dtype=np.float64)
        fl = (ctypes.c_double * 2)()
        _lib.call("cnb_chol_compliance", F._h, 3 * mo, colptr.ctypes.data, rowidx.ctypes.data, vals.ctypes.data,
                  U.data_ptr(), 3 * mo, fl, rank, world, _lib.stream())
        if world > 1:
            reduce_shards(U, group)
        if stats is not None:
            stats["fwd_flops"] = stats.get("fwd_flops", 0.0) + fl[0]
            stats["gram_flops"] = stats.get("gram_flops", 0.0) + fl[1]
    return ObjectCompliance(U=U, idx=torch.as_tensor(idx, device=d), side=torch.as_tensor(side, device=d),
                            full=full)
