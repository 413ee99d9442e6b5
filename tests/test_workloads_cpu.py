"""The bench-input generators (workloads.py) agree with the package's mesher."""

import numpy as np

import workloads
from paper_2306_06946_b200.mesh import five_tet_grid, surface_triangles


def test_five_tet_grid_identical():
    for shape, origin in (((4, 3, 5), (0.0, 0.0, 0.0)), ((7, 2, 3), (0.01, 0.2, -0.03))):
        nodes, tets = workloads.five_tet_grid(shape, 0.01, origin)
        mesh = five_tet_grid(shape, 0.01, origin)
        assert np.array_equal(nodes, mesh.nodes) and np.array_equal(tets, mesh.tets)
        assert np.array_equal(workloads.surface_triangles(tets), surface_triangles(mesh))


def test_cfg1_inputs_shapes():
    inp = workloads.cfg1_inputs()
    assert inp["nodes"].shape == (4000, 3)
    assert len(inp["Ds"]) == workloads.CFG1_REDRAWS and inp["Ds"][0].shape == (workloads.CFG1_CONTACTS, 3, 3)
    F = inp["Ds"][3]
    assert np.abs(np.einsum("gij,gkj->gik", F, F) - np.eye(3)).max() < 1e-14


def test_cfg4_generators_match_the_batched_scenes():
    from paper_2306_06946_b200 import batch

    n = 3 * 320
    a = workloads.cfg4_draws(5, 3, n)
    b = batch.cfg4_draws(5, 3, n)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    nodes, _ = workloads.five_tet_grid(workloads.CFG0_SHAPE, 0.01)
    nr = workloads.plane_normals(a[0])
    assert np.array_equal(nr, batch.plane_normals(a[0]))
    assert np.array_equal(workloads.placement(nodes, nr, 0.02), batch.placement(nodes, nr, 0.02))
