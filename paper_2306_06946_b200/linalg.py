"""Sparse symmetric storage, GPU supernodal Cholesky, solves, naive-order gemm.

Mirrors /root/reference/pkg/src/contactnewton/linalg.py: ``SparseSym``
(24-55), ``Factorization`` (58-106), ``factorize/solve/solve_multi``
(109-118), ``gemm`` (121-147).  The reference factorises with SuperLU on the
host; here ``Factorization`` runs a nested-dissection supernodal multifrontal
Cholesky whose symbolic analysis is host C++ (once per sparsity pattern) and
whose numeric factorisation and solves are sm_100a kernels (csrc/chol.cu).
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp
import torch

from . import _device as dv
from . import _lib
from .errors import DimensionMismatchError, NotSPDError

_SYM_RTOL = 1e-12


class SparsityPattern:
    """Immutable CSR pattern (host int64) plus optional node blocking / coordinates
    that steer the nested-dissection ordering."""

    def __init__(self, indptr, indices, n, block_size=1, coords=None):
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.n = int(n)
        self.block_size = int(block_size)
        self.coords = None if coords is None else np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])


class SparseSym:
    """Square symmetric sparse matrix: host CSR pattern + device fp64 values."""

    __slots__ = ("pattern", "values", "_csr_host")

    def __init__(self, mat=None, check: bool = True, *, pattern: SparsityPattern | None = None,
                 values: torch.Tensor | None = None):
        if pattern is not None:
            self.pattern = pattern
            self.values = values
            self._csr_host = None
            return
        if isinstance(mat, torch.Tensor):
            mat = mat.detach().cpu().numpy()
        csr = sp.csr_matrix(mat, dtype=np.float64)
        if csr.shape[0] != csr.shape[1]:
            raise DimensionMismatchError(f"matrix must be square, got {csr.shape}")
        csr.sum_duplicates()
        csr.sort_indices()
        if check:
            scale = max(np.abs(csr.data).max(initial=0.0), 1.0)
            asym = abs(csr - csr.T)
            if asym.nnz and asym.data.max() > _SYM_RTOL * scale:
                raise DimensionMismatchError(
                    f"matrix is not symmetric (max asymmetry {asym.data.max():.3e})")
        # the factorisation needs the symmetric pattern (both triangles)
        pat = (csr + csr.T).tocsr()
        pat.sort_indices()
        full = sp.csr_matrix((np.zeros(pat.nnz), pat.indices, pat.indptr), shape=csr.shape)
        full = (full + csr).tocsr()
        full.sort_indices()
        self.pattern = SparsityPattern(full.indptr, full.indices, csr.shape[0])
        self._csr_host = full
        self.values = None
        if torch.cuda.is_available():
            self.values = dv.f64(full.data)

    @property
    def dim(self) -> int:
        return self.pattern.n

    @classmethod
    def from_triplets(cls, dim, rows, cols, values, check: bool = True) -> "SparseSym":
        return cls(sp.coo_matrix((values, (rows, cols)), shape=(dim, dim)), check=check)

    @property
    def csr(self) -> sp.csr_matrix:
        vals = dv.host(self.values) if self.values is not None else self._csr_host.data
        return sp.csr_matrix((vals, self.pattern.indices, self.pattern.indptr),
                             shape=(self.dim, self.dim))

    def toarray(self) -> np.ndarray:
        return self.csr.toarray()

    def matvec(self, x):
        return self.csr @ dv.host(x)


class Factorization:
    """GPU Cholesky of a ``SparseSym``, reusable for many solves.

    ``solve_count`` counts back-solves like the reference (linalg.py:58-65);
    ``refactor(values)`` re-runs only the numeric phase on new values of the
    same pattern (corotational materials, once per step).
    """

    def __init__(self, matrix: SparseSym, leaf_nodes: int = 32):
        dev = _lib.require_cuda()
        pat = matrix.pattern
        self.dim = pat.n
        self.pattern = pat
        self.solve_count = 0
        handle = ctypes.c_void_p()
        coords = pat.coords
        _lib.check(_lib.lib().cnb_chol_analyze(
            pat.n, pat.indptr.ctypes.data, pat.indices.ctypes.data, pat.block_size,
            coords.ctypes.data if coords is not None else None, int(leaf_nodes), ctypes.byref(handle)),
            "chol_analyze")
        self._h = handle
        info = (ctypes.c_int64 * 9)()
        fl = (ctypes.c_double * 2)()
        _lib.call("cnb_chol_info", self._h, info, fl)
        self.n_supernodes = int(info[1])
        self.nnz_L = int(info[2])
        self.front_doubles = int(info[3])
        self.n_levels = int(info[4])
        self.flops = float(fl[0])
        self.solve_flops_per_rhs = float(fl[1])
        self._status = _lib.status(dev)
        self.refactor(matrix.values)

    def refactor(self, values: torch.Tensor) -> None:
        values = dv.f64(values)
        if values.numel() != self.pattern.nnz:
            raise DimensionMismatchError(
                f"values hold {values.numel()} entries, pattern has {self.pattern.nnz}")
        _lib.call("cnb_chol_factor", self._h, values.data_ptr(), self._status.ptr, _lib.stream())
        try:
            self._status.raise_if_set("factorize")
        except NotSPDError as exc:
            raise NotSPDError(f"{exc}; check masses, materials and time step") from None

    def refactor_async(self, values: torch.Tensor) -> None:
        """Numeric refactorisation without the host sync of the NotSPD check
        (the status word is checked at the next ``check_status``)."""
        _lib.call("cnb_chol_factor", self._h, values.data_ptr(), self._status.ptr, _lib.stream())

    def check_status(self) -> None:
        self._status.raise_if_set("factorize")

    def solve_device(self, B: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Solve for k right-hand sides given as a (k, n) contiguous device tensor."""
        k = B.shape[0]
        X = out if out is not None else torch.empty_like(B)
        _lib.call("cnb_chol_solve", self._h, B.data_ptr(), self.dim, X.data_ptr(), self.dim, k,
                  _lib.stream())
        return X

    def solve(self, b):
        b_t = dv.f64(b)
        if tuple(b_t.shape) != (self.dim,):
            raise DimensionMismatchError(f"rhs has shape {tuple(b_t.shape)}, expected ({self.dim},)")
        self.solve_count += 1
        return self.solve_device(b_t.reshape(1, -1)).reshape(-1)

    def solve_multi(self, B):
        B_t = dv.f64(B)
        if B_t.ndim != 2 or B_t.shape[0] != self.dim:
            raise DimensionMismatchError(
                f"rhs block has shape {tuple(B_t.shape)}, expected ({self.dim}, k)")
        self.solve_count += B_t.shape[1]
        return self.solve_device(B_t.t().contiguous()).t()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().cnb_chol_destroy(h)
            except Exception:
                pass
            self._h = None


def factorize(A: SparseSym) -> Factorization:
    return Factorization(A)


def solve(F: Factorization, b):
    return F.solve(b)


def solve_multi(F: Factorization, B):
    return F.solve_multi(B)


def gemm(A, B, transpose_a: bool = False, transpose_b: bool = False):
    """Dense product, ascending-k accumulation with separately rounded products and
    sums — bit-identical to the reference's naive gemm (linalg.py:121-147)."""
    A_t, B_t = dv.f64(A), dv.f64(B)
    if A_t.ndim != 2 or B_t.ndim != 2:
        raise DimensionMismatchError("gemm operands must be 2-d")
    m, k = (A_t.shape[1], A_t.shape[0]) if transpose_a else tuple(A_t.shape)
    kb, n = (B_t.shape[1], B_t.shape[0]) if transpose_b else tuple(B_t.shape)
    if k != kb:
        raise DimensionMismatchError(f"inner dimensions disagree: ({m}, {k}) x ({kb}, {n})")
    C = dv.empty((m, n))
    _lib.call("cnb_gemm_naive", m, n, k, A_t.data_ptr(), A_t.shape[1], int(transpose_a), B_t.data_ptr(),
              B_t.shape[1], int(transpose_b), C.data_ptr(), n, _lib.stream())
    return C
