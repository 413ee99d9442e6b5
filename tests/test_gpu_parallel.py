"""The multi-GPU column split of the compliance build (parallel.py,
cnb_chol_compliance_{plan,forward,gram,finish}) emulated on ONE GPU: the ranks'
phases run one after another in this process and each all-gather is a
concatenation in rank order.  No rank ever waits on another rank's kernel.
The gathered result must equal the single-GPU cnb_chol_compliance bit for bit
(every column's forward solve and every tile's Gram sum are computed exactly
as on one GPU), for E = unit columns (cfg1, barycentric contacts) and for
right-hand sides S^T directly (vertex contacts)."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_06946_b200 as m

    return m


def _single(F, k, colptr, rowidx, vals):
    from paper_2306_06946_b200 import _lib

    out = torch.empty((k, k), dtype=torch.float64, device="cuda")
    _lib.call("cnb_chol_compliance", F._h, k, colptr.ctypes.data, rowidx.ctypes.data, vals.ctypes.data,
              out.data_ptr(), k, None, _lib.stream())
    return out


def _emulated(F, k, colptr, rowidx, vals, world):
    from paper_2306_06946_b200.parallel import KernelSteps

    out = torch.full((k, k), float("nan"), dtype=torch.float64, device="cuda")
    steps = [KernelSteps(F, k, colptr, rowidx, vals, out, k, r, world) for r in range(world)]
    sends, cols = [], []
    for st in steps:
        send, ntile, _ = st.plan()
        y = torch.empty(send, dtype=torch.float64, device="cuda")
        st.forward(y)
        sends.append(y)
        cols.append(st.columns)
    yall = torch.cat(sends)
    tiles = []
    for st in steps:  # the plan lives in the handle: re-plan each rank before its gram
        send, ntile, _ = st.plan()
        t = torch.empty(ntile, dtype=torch.float64, device="cuda")
        st.gram(yall, t)
        tiles.append(t)
    steps[0].plan()
    steps[0].finish(torch.cat(tiles))
    # the column ranges tile [0, k) in rank order
    assert cols[0][0] == 0 and cols[-1][1] == k
    assert all(a[1] == b[0] for a, b in zip(cols, cols[1:]))
    return out


def _cfg1_columns(cn):
    import bench

    wl = bench.GpuWorkload(bench.make_inputs())
    csr = wl.S.sorted_csr
    dofs = np.unique(csr.indices).astype(np.int64)
    k = len(dofs)
    return wl.F, k, np.arange(k + 1, dtype=np.int64), dofs, np.ones(k)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_split_equals_single_gpu_unit_columns(cn, world):
    F, k, cp, ri, va = _cfg1_columns(cn)
    ref = _single(F, k, cp, ri, va)
    got = _emulated(F, k, cp, ri, va, world)
    assert torch.equal(got, ref)


def test_split_equals_single_gpu_signed_rows(cn, golden):
    g = golden("block_on_plane.npz")
    import scipy.sparse as sp

    import cn_oracle as orc

    E, nu, rho, a, b = g["mat0"]
    body = orc.Body(g["mesh0_nodes"], g["mesh0_tets"], young=E, poisson=nu, density=rho, alpha=a, beta=b)
    A, _ = body.system(g["mesh0_nodes"].ravel(), np.zeros(body.n), 0.01, (0.0, -9.81, 0.0))
    F = cn.Factorization(cn.SparseSym(A, check=False))
    # vertex rows: one unit entry per row, columns of S^T in CSC form
    rng = np.random.default_rng(3)
    verts = np.sort(rng.choice(len(g["mesh0_nodes"]), 70, replace=False))
    rows = (3 * verts[:, None] + np.arange(3)).ravel().astype(np.int64)
    k = len(rows)
    cp, va = np.arange(k + 1, dtype=np.int64), -np.ones(k)
    ref = _single(F, k, cp, rows, va)
    for world in (2, 4):
        assert torch.equal(_emulated(F, k, cp, rows, va, world), ref)
    S = sp.csr_matrix((va, (np.arange(k), rows)), shape=(k, body.n))
    dense = S @ orc.Factor(A).solve(S.T.toarray())
    assert np.abs(ref.cpu().numpy() - dense).max() <= 1e-9 * np.abs(dense).max()
