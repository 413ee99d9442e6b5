"""Constraint-space operators: directions, signed mapping, compliance, violation,
fast proximity update.

Mirrors /root/reference/pkg/src/contactnewton/constraints.py.  All dense
operators live on the GPU: ``rebuild_W_fast`` (3x3 block congruence,
bit-identical to the reference's naive gemm), ``compute_violation``,
``fast_update_proximity``, and ``assemble_Wg`` / ``assemble_W_standard``
(sparse-RHS forward solve on the supernodal factor + blocked Gram product,
csrc/solve.cu via wg.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _device as dv
from . import _lib
from .collision import DOF_KINDS, FrameSet, PairTable, attachment_triplets, frames_tensor
from .errors import DimensionMismatchError, InvalidAttachmentError


@dataclass
class DirectionMatrix:
    """Block-diagonal directions, (c_g, 3, 3) device tensor; block rows (n, t1, t2)."""

    blocks: torch.Tensor

    @property
    def n_groups(self) -> int:
        return int(self.blocks.shape[0])

    @property
    def c(self) -> int:
        return 3 * self.n_groups

    def as_dense(self) -> torch.Tensor:
        return torch.block_diag(*self.blocks) if self.n_groups else dv.zeros((0, 0))

    def as_sparse(self) -> sp.csr_matrix:
        if self.n_groups == 0:
            return sp.csr_matrix((0, 0))
        m = self.n_groups
        cols = (3 * np.arange(m)[:, None, None] + np.arange(3)[None, None, :]).repeat(3, axis=1)
        return sp.csr_matrix((dv.host(self.blocks).reshape(-1), cols.reshape(-1), np.arange(0, 9 * m + 1, 3)),
                             shape=(3 * m, 3 * m))

    def apply(self, rel) -> torch.Tensor:
        """D @ rel for a stacked (3p,) relative vector (constraints.py:58-60)."""
        rel_t = dv.f64(rel).reshape(-1, 3)
        out = dv.empty(self.c)
        zero = dv.zeros((self.n_groups, 3))
        _lib.call("cnb_violation", self.n_groups, self.blocks.data_ptr(), rel_t.data_ptr(), zero.data_ptr(),
                  out.data_ptr(), _lib.stream())
        return out

    def apply_transposed(self, lam, accumulate: torch.Tensor | None = None) -> torch.Tensor:
        """D^T @ lam (constraints.py:62-64); optionally also ``accumulate += D^T lam``."""
        lam_t = dv.f64(lam)
        out = dv.empty(self.c)
        _lib.call("cnb_apply_dt", self.n_groups, self.blocks.data_ptr(), lam_t.data_ptr(), out.data_ptr(),
                  accumulate.data_ptr() if accumulate is not None else None, _lib.stream())
        return out


def assemble_direction(frames) -> DirectionMatrix:
    """constraints.py:67-70."""
    return DirectionMatrix(frames_tensor(frames))


@dataclass
class Delassus:
    W: torch.Tensor

    @property
    def c(self) -> int:
        return int(self.W.shape[0])


@dataclass
class ObjectCompliance:
    """One object's S A^-1 S^T restricted to the pairs it takes part in.

    ``U`` is (3 mo x 3 mo) over pairs ``idx`` (ascending); ``side`` is +1 when the
    object owns side A of the pair, -1 for side B.  ``dense(dim)`` expands it to
    the reference's full (3p x 3p) per-object block (constraints.py:172-178).
    """

    U: torch.Tensor
    idx: torch.Tensor
    side: torch.Tensor
    full: bool  # idx == arange(p)

    def dense(self, dim: int) -> torch.Tensor:
        if self.full:
            return self.U
        out = dv.zeros((dim, dim))
        if len(self.idx):  # out = 0 + U at the object's rows (scatter-add kernel)
            _lib.call("cnb_scatter_add_compliance", int(self.idx.shape[0]), self.U.data_ptr(), self.U.shape[1],
                      self.idx.data_ptr(), out.data_ptr(), dim, _lib.stream())
        return out


@dataclass
class MappingDelassus:
    """W_g = sum_o S_o A_o^-1 S_o^T (3p x 3p) plus the per-object parts."""

    wg: torch.Tensor
    per_object: dict

    @property
    def dim(self) -> int:
        return int(self.wg.shape[0])


@dataclass
class SignedMapping:
    """S_o for one object: host CSR (3p x n_o) and the device CSR of S_o^T used by the
    mechanical correction; ``idx``/``side`` give the object's pair participation."""

    csr: sp.csr_matrix
    idx: np.ndarray
    side: np.ndarray
    _dev: tuple | None = None
    _sorted: sp.csr_matrix | None = None

    @property
    def sorted_csr(self) -> sp.csr_matrix:
        """The same matrix with ascending columns per row (device planning order);
        ``csr`` keeps the reference's own entry order."""
        if self._sorted is None:
            self._sorted = self.csr.sorted_indices() if not self.csr.has_sorted_indices else self.csr
        return self._sorted

    @property
    def shape(self):
        return self.csr.shape

    @property
    def nnz(self):
        return self.csr.nnz

    @property
    def T(self):
        return self.csr.T

    def toarray(self):
        return self.csr.toarray()

    def device_transpose(self):
        """(rowptr, col, val) of S^T on the device, cached."""
        if self._dev is None:
            st = self.csr.T.tocsr()
            st.sort_indices()
            d = dv.device()
            self._dev = (dv.upload(st.indptr.astype(np.int64)),
                         dv.upload(st.indices.astype(np.int64)), dv.f64(st.data, d))
        return self._dev

    def rmatvec(self, t: torch.Tensor, out: torch.Tensor | None = None, alpha: float = 1.0) -> torch.Tensor:
        """out = alpha * S^T t on the device (deterministic row-gather SpMV)."""
        rp, ci, va = self.device_transpose()
        n = self.csr.shape[1]
        y = out if out is not None else dv.empty(n)
        _lib.call("cnb_csr_spmv", n, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), t.data_ptr(), y.data_ptr(),
                  float(alpha), _lib.stream())
        return y


def build_signed_mapping(pairs, object_id: int, n_dofs: int, fixed_mask=None) -> SignedMapping:
    """+G on A sides, -G on B sides, fixed-DOF columns zeroed (constraints.py:101-120)."""
    if isinstance(pairs, PairTable) and not (pairs.h_kind == 2).any():
        return _signed_mapping_table(pairs, object_id, n_dofs, fixed_mask)
    plist = pairs.pairs if isinstance(pairs, PairTable) else list(pairs)
    rows, cols, vals = [], [], []
    idx, side = [], []
    for i, pair in enumerate(plist):
        for attach, sign in ((pair.attach_a, 1.0), (pair.attach_b, -1.0)):
            if attach.object_id != object_id or attach.kind not in DOF_KINDS:
                continue
            r, c, v = attachment_triplets(attach, n_dofs, 3 * i)
            rows += r
            cols += c
            vals += [sign * x for x in v]
            idx.append(i)
            side.append(1 if sign > 0 else -1)
    S = sp.coo_matrix((vals, (rows, cols)), shape=(3 * len(plist), n_dofs)).tocsr()
    if fixed_mask is not None and np.asarray(fixed_mask).any():
        # the reference's product keeps its (unsorted) column order per row
        S = (S @ sp.diags(np.where(fixed_mask, 0.0, 1.0))).tocsr()
    return SignedMapping(S, np.asarray(idx, dtype=np.int64), np.asarray(side, dtype=np.int8))


def _signed_mapping_table(table: PairTable, object_id: int, n_dofs: int, fixed_mask=None) -> SignedMapping:
    """build_signed_mapping from the table arrays (vertex / barycentric sides): the
    same triplets as attachment_triplets, pair by pair, side A before side B."""
    m = table.m
    kind, obj, node, w = table.h_kind, table.h_obj, table.h_node, table.h_w
    mine = (obj == object_id) & ((kind == 0) | (kind == 1))          # (m, 2)
    ii, ss = np.nonzero(mine)                                        # row-major: pair, then side
    nn = np.where(kind[ii, ss] == 0, 1, 3)
    cols_node = node[ii, ss]                                         # (k, 3)
    used = np.arange(3)[None, :] < nn[:, None]
    if (used & ((cols_node < 0) | (3 * cols_node + 2 >= n_dofs))).any():
        raise InvalidAttachmentError("attachment node out of range")
    sign = np.where(ss == 0, 1.0, -1.0)
    rows, cols, vals = [], [], []
    for j in range(3):  # node j of each attachment
        sel = j < nn
        for a in range(3):
            rows.append(3 * ii[sel] + a)
            cols.append(3 * cols_node[sel, j] + a)
            vals.append(sign[sel] * w[ii[sel], ss[sel], j])
    rows = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    cols = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    vals = np.concatenate(vals) if vals else np.zeros(0)
    S = sp.coo_matrix((vals, (rows, cols)), shape=(3 * m, n_dofs)).tocsr()
    if fixed_mask is not None and np.asarray(fixed_mask).any():
        # same CSR as the reference before the product, so the same (unsorted)
        # column order per row after it (constraints.py:116-119)
        S = (S @ sp.diags(np.where(fixed_mask, 0.0, 1.0))).tocsr()
    return SignedMapping(S, ii.astype(np.int64), np.where(ss == 0, 1, -1).astype(np.int8))


def assemble_H(D: DirectionMatrix, G) -> sp.csr_matrix:
    """H = D G (constraints.py:123-129); host sparse (standard scheme / verification)."""
    Gm = G.csr if isinstance(G, SignedMapping) else G
    if D.c != Gm.shape[0]:
        raise DimensionMismatchError(
            f"direction matrix acts on {D.c} proximity rows, mapping has {Gm.shape[0]}")
    return (D.as_sparse() @ Gm).tocsr()


def _as_mapping(G) -> SignedMapping:
    """Wrap a host CSR (3p x n) as a SignedMapping; participation = pairs with stored rows."""
    if isinstance(G, SignedMapping):
        return G
    csr = sp.csr_matrix(G)
    csr.sort_indices()
    nz = np.diff(csr.indptr).reshape(-1, 3).sum(axis=1) > 0 if csr.shape[0] else np.zeros(0, bool)
    idx = np.flatnonzero(nz).astype(np.int64)
    return SignedMapping(csr, idx, np.ones(len(idx), dtype=np.int8))


def _sum_compliance(parts: list, dim: int) -> torch.Tensor:
    """sum_o of the per-object parts expanded to dim x dim, ascending object id."""
    if not parts:
        return dv.zeros((dim, dim))
    total = None
    for comp in parts:
        if total is None:
            total = comp.dense(dim).clone() if len(parts) > 1 else comp.dense(dim)
        elif comp.full:
            total += comp.U
        elif len(comp.idx):
            mo = int(comp.idx.shape[0])
            _lib.call("cnb_scatter_add_compliance", mo, comp.U.data_ptr(), comp.U.shape[1], comp.idx.data_ptr(),
                      total.data_ptr(), total.shape[1], _lib.stream())
    return total


def assemble_W_standard(H_by_object: dict, F_by_object: dict, group=None) -> Delassus:
    """W = sum_o H_o A_o^-1 H_o^T (constraints.py:132-152).

    The reference forms X = A^-1 H^T with a dense multi-RHS solve and multiplies
    by H; here H^T's columns go through the same sparse-RHS forward solve + Gram
    product as W_g (wg.py), since H_o = D S_o has S_o's sparsity per pair.
    """
    from .wg import object_compliance

    ids = sorted(H_by_object)
    if not ids:
        return Delassus(dv.zeros((0, 0)))
    c = H_by_object[ids[0]].shape[0]
    parts = []
    for oid in ids:
        H = _as_mapping(H_by_object[oid])
        F = F_by_object[oid]
        if H.shape[1] != F.dim:
            raise DimensionMismatchError(f"object {oid}: H has {H.shape[1]} columns, factorization dim {F.dim}")
        parts.append(object_compliance(H, F, c, group=group))
    return Delassus(_sum_compliance(parts, c))


def assemble_Wg(S_by_object: dict, F_by_object: dict, group=None) -> MappingDelassus:
    """W_g = sum_o S_o A_o^-1 S_o^T and the per-object parts (constraints.py:155-179).

    Per object: Y = L^-1 P S^T by a sparse-RHS forward solve over the supernodal
    tree, then U = Y^T Y by a blocked Gram product (fp64 MMA) restricted to the
    supernodes each column's elimination path touches.  Objects are summed in
    ascending id order like the reference.
    """
    from .wg import object_compliance

    ids = sorted(S_by_object)
    if not ids:
        return MappingDelassus(dv.zeros((0, 0)), {})
    dim = S_by_object[ids[0]].shape[0]
    per = {}
    for oid in ids:
        S = S_by_object[oid]
        F = F_by_object[oid]
        if S.shape[1] != F.dim:
            raise DimensionMismatchError(f"object {oid}: S has {S.shape[1]} columns, factorization dim {F.dim}")
        per[oid] = object_compliance(S, F, dim, group=group)
    return MappingDelassus(_sum_compliance([per[o] for o in ids], dim), per)


def sum_compliance(per: dict, dim: int) -> MappingDelassus:
    """W_g from per-object parts already formed (object_compliance), summed in
    ascending object id like assemble_Wg."""
    return MappingDelassus(_sum_compliance([per[o] for o in sorted(per)], dim), per)


def rebuild_W_fast(D: DirectionMatrix, wg: MappingDelassus, out: torch.Tensor | None = None) -> Delassus:
    """W = D W_g D^T (constraints.py:182-191), bit-identical to the reference."""
    if D.c != wg.dim:
        raise DimensionMismatchError(f"direction matrix is {D.c} rows, W_g is {wg.dim}")
    W = out if out is not None else dv.square(D.c)
    if D.c:
        _lib.call("cnb_rebuild_w", D.n_groups, D.blocks.data_ptr(), wg.wg.data_ptr(), dv.ld(wg.wg),
                  W.data_ptr(), dv.ld(W), _lib.stream())
    return Delassus(W)


@dataclass
class Violation:
    delta: torch.Tensor

    def normal_components(self) -> torch.Tensor:
        return self.delta.reshape(-1, 3)[:, 0]

    def max_penetration(self) -> float:
        n = self.normal_components()
        return float(max(0.0, -(float(n.min()) if n.numel() else 0.0)))


def compute_violation(D: DirectionMatrix, p_a, p_b, out: torch.Tensor | None = None) -> Violation:
    """delta = D (p_a - p_b) (constraints.py:208-214)."""
    pa, pb = dv.f64(p_a), dv.f64(p_b)
    if pa.numel() != D.c:
        raise DimensionMismatchError(f"positions stack to {pa.numel()}, direction matrix expects {D.c}")
    delta = out if out is not None else dv.empty(D.c)
    if D.c:
        _lib.call("cnb_violation", D.n_groups, D.blocks.data_ptr(), pa.data_ptr(), pb.data_ptr(),
                  delta.data_ptr(), _lib.stream())
    return Violation(delta)


def prox_update_inplace(p_a: torch.Tensor, p_b: torch.Tensor, wg: MappingDelassus, t: torch.Tensor,
                        h: float) -> None:
    """p_a / p_b += / -= h^2 U_o t for every dynamic object (device, in place)."""
    for oid in sorted(wg.per_object):
        comp = wg.per_object[oid]
        mo = int(comp.idx.shape[0])
        if mo == 0:
            continue
        _lib.call("cnb_prox_update", mo, comp.U.data_ptr(), comp.U.shape[1],
                  None if comp.full else comp.idx.data_ptr(), comp.side.data_ptr(), t.data_ptr(), float(h),
                  p_a.data_ptr(), p_b.data_ptr(), _lib.stream())


def fast_update_proximity(p_a, p_b, wg: MappingDelassus, D: DirectionMatrix, lam, h: float, pairs):
    """Proximity positions after one corrective impulse, no system solves
    (constraints.py:217-244).  Returns new tensors; inputs are not modified."""
    lam_t = dv.f64(lam)
    if tuple(lam_t.shape) != (D.c,):
        raise DimensionMismatchError(f"lambda has shape {tuple(lam_t.shape)}, expected ({D.c},)")
    t = D.apply_transposed(lam_t)
    pa = dv.f64(p_a).reshape(-1, 3).clone()
    pb = dv.f64(p_b).reshape(-1, 3).clone()
    prox_update_inplace(pa, pb, wg, t, h)
    return pa, pb
