"""Per-object mapping compliance U_o = S_o A_o^-1 S_o^T on the GPU factor.

Replaces the multi-RHS solve + sparse product of assemble_Wg
(/root/reference/pkg/src/contactnewton/constraints.py:175-178): instead of
X = A^-1 S^T (n x 3p dense) and S X, the library forward-solves only the
elimination paths of the right-hand sides (Y = L^-1 P R) and forms Y^T Y with
fp64 tensor-core tiles (csrc/solve.cu: panel_mma_kernel, gram_kernel).  Only
the rows/columns of the pairs the object takes part in are formed.

Right-hand sides: when the rows of S_o touch fewer distinct DoFs k than they
are (barycentric contacts share triangle nodes, a node can carry several
pairs), R = E, the unit columns of those k DoFs: C = E^T A^-1 E (k x k) and
U_o = S_o C S_o^T (csrc/contact.cu sandwich_kernel).  Same matrix, k^2
instead of (3 m_o)^2 Gram work.  Otherwise R = S_o^T directly.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as dv
from . import _lib


DOF_REDUCTION_MAX = 0.85  # use the DoF-reduced right-hand sides when k <= 0.85 * 3 m_o
ELL_WIDTH = 4             # nnz per row of S_o the sandwich kernel takes (barycentric: 3)
SANDWICH_MAX_K = 29000    # row buffer of the sandwich kernel (227 KB of shared memory)


def object_compliance(S, F, dim: int, stats: dict | None = None, group=None, shard: bool = True):
    """U_o for one object.  Under torch.distributed (world > 1) the right-hand-side
    columns are split across ranks (forward solve + Gram tiles) and joined by two
    NCCL all-gathers (parallel.split_compliance); the result is bit-identical."""
    from .constraints import ObjectCompliance
    from .parallel import split_compliance, world_info

    rank, world = world_info(group) if shard else (0, 1)

    idx, side = S.idx, S.side
    mo = len(idx)
    d = dv.device()
    full = mo == dim // 3 and (mo == 0 or np.array_equal(idx, np.arange(mo)))
    U = dv.empty((3 * mo, 3 * mo))
    if mo:
        rows = (3 * idx[:, None] + np.arange(3)).ravel()
        csr = S.sorted_csr
        colptr = np.zeros(3 * mo + 1, dtype=np.int64)
        counts = np.diff(csr.indptr)[rows]
        colptr[1:] = np.cumsum(counts)
        starts = csr.indptr[rows]
        # the CSR entries of those rows, row by row (vectorised ranges)
        sel = np.repeat(starts - colptr[:-1], counts) + np.arange(colptr[-1], dtype=np.int64)
        rowidx = np.ascontiguousarray(csr.indices[sel], dtype=np.int64)
        vals = np.ascontiguousarray(csr.data[sel], dtype=np.float64)
        fl = (ctypes.c_double * 2)()
        dofs, inv = np.unique(rowidx, return_inverse=True)
        k = len(dofs)
        per_row = np.diff(colptr)
        if k <= DOF_REDUCTION_MAX * 3 * mo and per_row.max(initial=0) <= ELL_WIDTH and k <= SANDWICH_MAX_K:
            # C = E^T A^-1 E over the k touched DoFs, then U = S C S^T
            e_ptr = np.arange(k + 1, dtype=np.int64)
            e_val = np.ones(k)
            dofs = np.ascontiguousarray(dofs, dtype=np.int64)
            C = dv.empty((k, k))
            if world > 1:
                info = split_compliance(F, k, e_ptr, dofs, e_val, C, k, group=group, rank=rank, world=world)
                fl[0], fl[1] = info["flops"]
            else:
                _lib.call("cnb_chol_compliance", F._h, k, e_ptr.ctypes.data, dofs.ctypes.data, e_val.ctypes.data,
                          C.data_ptr(), k, fl, _lib.stream())
            ell_col = np.zeros((3 * mo, ELL_WIDTH), dtype=np.int32)
            ell_val = np.zeros((3 * mo, ELL_WIDTH))
            slot = np.arange(len(rowidx)) - np.repeat(colptr[:-1], per_row)
            rix = np.repeat(np.arange(3 * mo), per_row)
            ell_col[rix, slot] = inv
            ell_val[rix, slot] = vals
            d_col = dv.upload(ell_col)
            d_val = dv.upload(ell_val)
            _lib.call("cnb_sandwich", 3 * mo, k, d_col.data_ptr(), d_val.data_ptr(), C.data_ptr(), k, U.data_ptr(),
                      3 * mo, _lib.stream())
        elif world > 1:
            info = split_compliance(F, 3 * mo, colptr, rowidx, vals, U, 3 * mo, group=group, rank=rank, world=world)
            fl[0], fl[1] = info["flops"]
        else:
            _lib.call("cnb_chol_compliance", F._h, 3 * mo, colptr.ctypes.data, rowidx.ctypes.data, vals.ctypes.data,
                      U.data_ptr(), 3 * mo, fl, _lib.stream())
        if stats is not None:
            stats["fwd_flops"] = stats.get("fwd_flops", 0.0) + fl[0]
            stats["gram_flops"] = stats.get("gram_flops", 0.0) + fl[1]
    return ObjectCompliance(U=U, idx=dv.upload(idx), side=dv.upload(side), full=full)
