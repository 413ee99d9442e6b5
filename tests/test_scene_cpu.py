"""Host-side scene logic without a GPU: the Newton iteration count a step
without contacts reports, as the reference's loop (solver.py:260-367) counts
it on empty pairs (StepReport.newton_iterations = len(result.iterations),
scene.py:744)."""

from paper_2306_06946_b200.scene import _contactless_iterations
from paper_2306_06946_b200.solver import NewtonConfig


def test_contactless_iteration_counts():
    # defaults: pen 0 <= 1e-5 stops after the first iteration
    assert len(_contactless_iterations(NewtonConfig(scheme="fast", max_iterations=5))) == 1
    # forced iterations: every iteration runs an empty PGS
    forced = NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0, rotation_tol=-1.0)
    its = _contactless_iterations(forced)
    assert len(its) == 5 and all(i.pgs_iterations == 0 and i.penetration == 0.0 for i in its)
    # forced penetration, default rotation tolerance: the zero rotation stops iteration 2
    assert len(_contactless_iterations(NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0))) == 1
    # no re-linearisation: only the penetration test stops the loop
    nr = NewtonConfig(scheme="standard", max_iterations=4, penetration_tol=-1.0, relinearize=False)
    assert len(_contactless_iterations(nr)) == 4
    assert len(_contactless_iterations(NewtonConfig(scheme="single", max_iterations=7, penetration_tol=-1.0))) == 1


def test_colour_groups_separates_shared_dofs():
    """colour_groups (coloured PGS option): a partition of the groups in which no
    two groups touching the same node of an object share a colour, each colour
    in canonical order, greedy in canonical order."""
    import numpy as np
    import scipy.sparse as sp

    from paper_2306_06946_b200.solver import colour_groups

    rng = np.random.default_rng(0)
    m, nn = 60, 40
    rows, cols = [], []
    for i in range(m):
        for node in rng.choice(nn, 3, replace=False):
            for a in range(3):
                rows.append(3 * i + a)
                cols.append(3 * node + a)
    S0 = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(3 * m, 3 * nn))
    S1 = sp.csr_matrix((np.ones(m * 3), (np.arange(3 * m), np.arange(3 * m) % 9)), shape=(3 * m, 9))
    ptr, grp = colour_groups({0: S0, 1: S1}, m)
    assert ptr[0] == 0 and ptr[-1] == m and np.array_equal(np.sort(grp), np.arange(m))
    colour = np.empty(m, dtype=int)
    for k in range(len(ptr) - 1):
        members = grp[ptr[k]:ptr[k + 1]]
        assert np.all(np.diff(members) > 0)
        colour[members] = k
    nodes0 = [set(S0.indices[S0.indptr[3 * i]:S0.indptr[3 * i + 3]] // 3) for i in range(m)]
    nodes1 = [set(S1.indices[S1.indptr[3 * i]:S1.indptr[3 * i + 3]] // 3) for i in range(m)]
    for i in range(m):
        for j in range(i):
            if nodes0[i] & nodes0[j] or nodes1[i] & nodes1[j]:
                assert colour[i] != colour[j]
    assert colour[0] == 0
