"""CPU checks of the host symbolic analysis (csrc/symbolic.cpp).

The analysis is host C++, so it runs here without a GPU.  A numpy emulation
of the multifrontal numeric phase walks the exported structure (fronts,
extend-add maps, value map, levels) exactly as the CUDA kernels do; its
solution must match scipy's direct solve.  This pins the symbolic layer
before any GPU time is spent.
"""

import ctypes

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import cn_oracle as orc
from paper_2306_06946_b200 import _lib
from paper_2306_06946_b200.mesh import box_mesh, five_tet_grid


def analyze(A, bs=1, coords=None, leaf=8):
    A = sp.csr_matrix(A)
    A.sort_indices()
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(A.indices, dtype=np.int64)
    h = ctypes.c_void_p()
    c = None if coords is None else np.ascontiguousarray(coords, dtype=np.float64)
    _lib.check(_lib.lib().cnb_chol_analyze(A.shape[0], indptr.ctypes.data, indices.ctypes.data, bs,
                                           c.ctypes.data if c is not None else None, leaf, ctypes.byref(h)))
    info = (ctypes.c_int64 * 9)()
    fl = (ctypes.c_double * 2)()
    _lib.call("cnb_chol_info", h, info, fl)
    out = {"info": list(info), "flops": fl[0]}
    dtypes = {"rel": np.int32, "level": np.int32}
    for name in ("perm", "iperm", "first", "rows_ptr", "rows", "parent", "level", "child_ptr", "child",
                 "front_off", "rel_ptr", "rel", "map_src", "map_dst", "level_ptr", "level_sn"):
        nb = _lib.lib().cnb_chol_export_bytes(h, name.encode())
        arr = np.empty(nb // np.dtype(dtypes.get(name, np.int64)).itemsize, dtype=dtypes.get(name, np.int64))
        _lib.call("cnb_chol_export", h, name.encode(), arr.ctypes.data)
        out[name] = arr
    _lib.lib().cnb_chol_destroy(h)
    return out, A


def emulate_factor_solve(S, A, b):
    ns = len(S["first"]) - 1
    nc = np.diff(S["first"])
    nr = np.diff(S["rows_ptr"])
    f = nc + nr
    ldf = f + (f & 1)  # front columns are stored with an even stride (16-byte aligned)
    assert np.array_equal(np.diff(S["front_off"]), ldf * f)
    fronts = np.zeros(S["front_off"][-1])
    fronts[S["map_dst"]] = A.data[S["map_src"]]
    F = [fronts[S["front_off"][s]:S["front_off"][s + 1]].reshape(f[s], ldf[s])[:, :f[s]].T.copy() for s in range(ns)]
    children = [S["child"][S["child_ptr"][s]:S["child_ptr"][s + 1]] for s in range(ns)]
    rel = [S["rel"][S["rel_ptr"][s]:S["rel_ptr"][s + 1]] for s in range(ns)]
    for l in range(len(S["level_ptr"]) - 1):
        for s in S["level_sn"][S["level_ptr"][l]:S["level_ptr"][l + 1]]:
            for c in children[s]:
                U = np.tril(F[c][nc[c]:, nc[c]:])
                F[s][np.ix_(rel[c], rel[c])] += U
            k = nc[s]
            Fs = np.tril(F[s])
            L11 = np.linalg.cholesky(Fs[:k, :k])
            L21 = np.linalg.solve(L11, Fs[k:, :k].T).T
            F[s][:k, :k] = L11
            F[s][k:, :k] = L21
            F[s][k:, k:] = Fs[k:, k:] - L21 @ L21.T
    # solve with the permutation
    n = A.shape[0]
    y = b[S["perm"]].copy()
    for s in range(ns):  # postorder: children first
        a, e = S["first"][s], S["first"][s + 1]
        rows = S["rows"][S["rows_ptr"][s]:S["rows_ptr"][s + 1]]
        L11 = F[s][:nc[s], :nc[s]]
        ys = np.linalg.solve(np.tril(L11), y[a:e])
        y[a:e] = ys
        y[rows] -= F[s][nc[s]:, :nc[s]] @ ys
    x = y
    for s in range(ns - 1, -1, -1):
        a, e = S["first"][s], S["first"][s + 1]
        rows = S["rows"][S["rows_ptr"][s]:S["rows_ptr"][s + 1]]
        r = x[a:e] - F[s][nc[s]:, :nc[s]].T @ x[rows]
        x[a:e] = np.linalg.solve(np.tril(F[s][:nc[s], :nc[s]]).T, r)
    out = np.empty(n)
    out[S["perm"]] = x
    return out


def _check(A, bs=1, coords=None, leaf=8):
    S, A = analyze(A, bs, coords, leaf)
    n = A.shape[0]
    assert np.array_equal(np.sort(S["perm"]), np.arange(n))
    assert np.array_equal(S["iperm"][S["perm"]], np.arange(n))
    # every lower entry of P A P^T is mapped exactly once, to distinct slots
    Ap = A[S["perm"]][:, S["perm"]]
    assert len(S["map_src"]) == sp.tril(Ap).nnz
    assert len(np.unique(S["map_dst"])) == len(S["map_dst"])
    b = np.random.default_rng(0).standard_normal(n)
    x = emulate_factor_solve(S, A, b)
    ref = spla.spsolve(A.tocsc(), b)
    assert np.abs(x - ref).max() <= 1e-10 * np.abs(ref).max()
    return S


def test_random_spd_graph_ordering():
    rng = np.random.default_rng(1)
    n = 60
    M = sp.random(n, n, density=0.08, random_state=3)
    A = (M @ M.T + sp.eye(n) * n).tocsr()
    _check(A, bs=1, leaf=4)


def test_fe_block_geometric_ordering():
    mesh = five_tet_grid((6, 4, 5), 0.01)
    body = orc.Body(mesh.nodes, mesh.tets, young=5e3, poisson=0.45, fixed_nodes=[0, 1, 2])
    A, _ = body.system(mesh.nodes.ravel(), np.zeros(3 * mesh.n_nodes), 0.01, (0, -9.81, 0))
    S = _check(A, bs=3, coords=mesh.nodes, leaf=8)
    assert S["info"][1] > 1  # more than one supernode


def test_kuhn_box_graph_ordering():
    mesh = box_mesh((0.1, 0.1, 0.1), (3, 3, 3))
    body = orc.Body(mesh.nodes, mesh.tets)
    A, _ = body.system(mesh.nodes.ravel(), np.zeros(3 * mesh.n_nodes), 0.01, (0, -9.81, 0))
    _check(A, bs=3, coords=None, leaf=6)


def test_fill_is_reasonable_against_superlu():
    mesh = five_tet_grid((20, 10, 10), 0.01)
    body = orc.Body(mesh.nodes, mesh.tets, young=5e3, poisson=0.45)
    A, _ = body.system(mesh.nodes.ravel(), np.zeros(3 * mesh.n_nodes), 0.01, (0, -9.81, 0))
    S, _ = analyze(A, bs=3, coords=mesh.nodes, leaf=32)
    lu = spla.splu(A.tocsc(), permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                   options=dict(SymmetricMode=True))
    nnz_superlu = lu.L.nnz
    # stored entries include structural zeros of relaxed supernodes; plain
    # nested dissection fills more than minimum degree at this small size
    assert S["info"][2] <= 3.0 * nnz_superlu, (S["info"][2], nnz_superlu)


def test_reference_matrix_with_fixed_nodes(golden):
    """The reference's own A (fixed nodes [0, 1, 2]: identity rows, the fixed
    nodes isolated in the node graph) through the blocked geometric analysis."""
    g = golden("kat_linalg.npz")
    n = len(g["b"])
    A = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    S, A = analyze(A, bs=3, coords=g["nodes"], leaf=4)
    x = emulate_factor_solve(S, A, g["b"])
    assert np.abs(x - g["x"]).max() <= 1e-12 * np.abs(g["x"]).max()
