"""Integer patterns of the system matrix A against the reference (CPU, no GPU).

SoftBody.assemble (reference dynamics.py:183-211) keeps a stiffness entry only
when neither its row nor its column is a fixed DoF and adds one diagonal entry
per DoF (190-200); structural zeros of the kept 3x3 blocks stay.  The layout
that drives the device assembly (``_FeLayout``) must produce exactly that
pattern: the fixtures were written by the reference (tests/golden/make_golden.py).
"""

import numpy as np

from paper_2306_06946_b200.dynamics import _FeLayout


def _fixed_dofs(n_nodes, fixed_nodes):
    mask = np.zeros(3 * n_nodes, dtype=bool)
    for k in fixed_nodes:
        mask[3 * k:3 * k + 3] = True
    return mask


def test_stiffness_and_system_pattern_kat_linalg(golden):
    g = golden("kat_linalg.npz")
    nn = len(g["nodes"])
    lay = _FeLayout(nn, g["tets"])
    # K: full node adjacency in 3x3 blocks
    assert np.array_equal(lay.rowptr, g["K_indptr"])
    assert np.array_equal(lay.indices, g["K_indices"])
    rowptr, indices, src = lay.system_pattern(_fixed_dofs(nn, [0, 1, 2]))
    assert np.array_equal(rowptr, g["indptr"])
    assert np.array_equal(indices, g["indices"])
    # src points at K entries with the same (row, col); fixed diagonals are -1
    krow = np.repeat(np.arange(3 * nn), np.diff(lay.rowptr))
    arow = np.repeat(np.arange(3 * nn), np.diff(rowptr))
    kept = src >= 0
    assert np.array_equal(krow[src[kept]], arow[kept])
    assert np.array_equal(lay.indices[src[kept]], indices[kept])
    assert np.array_equal(arow[~kept], indices[~kept])
    assert (~kept).sum() == 9


def test_system_pattern_two_bodies_with_fixed_nodes(golden):
    g = golden("fixed_mapping.npz")
    for oid, name, fixed in ((0, "lower", g["fixed"]), (1, "upper", [])):
        nodes, tets = g[f"{name}_nodes"], g[f"{name}_tets"]
        lay = _FeLayout(len(nodes), tets)
        rowptr, indices, src = lay.system_pattern(_fixed_dofs(len(nodes), fixed))
        assert np.array_equal(rowptr, g[f"A{oid}_indptr"])
        assert np.array_equal(indices, g[f"A{oid}_indices"])
        assert (src is None) == (len(fixed) == 0)


def test_system_pattern_no_fixed_shares_stiffness_pattern(golden):
    g = golden("kat_linalg.npz")
    lay = _FeLayout(len(g["nodes"]), g["tets"])
    rowptr, indices, src = lay.system_pattern(np.zeros(3 * len(g["nodes"]), dtype=bool))
    assert src is None and rowptr is lay.rowptr and indices is lay.indices
