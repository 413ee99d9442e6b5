"""Bit-exact integer patterns through the product path against reference-written
fixtures: the system matrix returned by SoftBody.assemble (reference
dynamics.py:183-211, fixed rows/cols dropped at 190-200) and the signed mapping
S_o built inside Simulation.prepare_step (constraints.py:101-120, fixed columns
zeroed), plus a 3-step trajectory of a scene whose contacts land on fixed DoFs."""

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


def _h(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _rel(a, b):
    a, b = _h(a), _h(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_soft_body_assemble_pattern_kat_linalg(cn, golden):
    g = golden("kat_linalg.npz")
    body = cn.SoftBody(cn.TetMesh(g["nodes"], g["tets"]), young=5e4, poisson=0.3, fixed_nodes=np.array([0, 1, 2]))
    st = cn.MechanicalState(g["q"], g["v"])
    A, b = body.assemble(st, 0.01, (0.0, -9.81, 0.0))
    csr = A.csr
    assert np.array_equal(csr.indptr, g["indptr"])
    assert np.array_equal(csr.indices, g["indices"])
    assert _rel(csr.data, g["data"]) <= 1e-12
    assert _rel(b, g["b"]) <= 1e-12
    F = cn.factorize(A)
    assert _rel(F.solve(b), g["x"]) <= 1e-12


def _fixed_scene(cn, g):
    lower = cn.SoftSpec(name="lower", mesh=cn.TetMesh(g["lower_nodes"], g["lower_tets"]), young=1e4, poisson=0.4,
                        density=1000.0, fixed_nodes=g["fixed"])
    upper = cn.SoftSpec(name="upper", mesh=cn.TetMesh(g["upper_nodes"], g["upper_tets"]), young=2e3, poisson=0.4,
                        density=1000.0, velocity=(0.0, -0.1, 0.0))
    plane = cn.PlaneSpec(name="ground", normal=(0.0, 1.0, 0.0), offset=0.0)
    return cn.SceneConfig(objects=[lower, upper, plane], h=0.01, threshold=0.004,
                          pgs=cn.PgsConfig(max_iterations=400, tolerance=1e-10, friction=0.4),
                          newton=cn.NewtonConfig(scheme="fast", max_iterations=3, penetration_tol=-1.0,
                                                 rotation_tol=-1.0),
                          output=cn.OutputConfig(snapshots=False, metrics=False))


def test_signed_mapping_and_system_patterns_with_fixed_dofs(cn, golden):
    g = golden("fixed_mapping.npz")
    sim = cn.Simulation(_fixed_scene(cn, g))
    ctx = sim.prepare_step(build_wg=True)[0]
    keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in ctx.pairs])
    assert np.array_equal(keys, g["s0_keys"])
    for oid in (0, 1):
        S = ctx.S_by_object[oid].csr
        assert np.array_equal(S.indptr, g[f"S{oid}_indptr"])
        assert np.array_equal(S.indices, g[f"S{oid}_indices"])
        assert np.array_equal(S.data, g[f"S{oid}_data"])
        obj = sim.objects[oid]
        A, b = obj.body.assemble(obj.state, 0.01, (0.0, -9.81, 0.0))
        assert np.array_equal(A.csr.indptr, g[f"A{oid}_indptr"])
        assert np.array_equal(A.csr.indices, g[f"A{oid}_indices"])
        assert _rel(A.csr.data, g[f"A{oid}_data"]) <= 1e-12
        assert _rel(b, g[f"b{oid}"]) <= 1e-12


def test_fixed_mapping_trajectory(cn, golden):
    g = golden("fixed_mapping.npz")
    sim = cn.Simulation(_fixed_scene(cn, g))
    for s in range(3):
        rep = sim.step()
        assert rep.c_groups == int(g[f"s{s}_npairs"])
        assert rep.newton_iterations == int(g[f"s{s}_newton"])
        if s == 0:
            keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in sim.last_pairs])
            assert np.array_equal(keys, g["s0_keys"])
            lh = _h(torch.stack(sim.last_result.lam_history))
            assert np.abs(lh - g["s0_lamhist"]).max() <= 1e-6 * max(np.abs(g["s0_lamhist"]).max(), 1e-300)
        for o in (0, 1):
            q = g[f"s{s}_q{o}"]
            assert np.abs(_h(sim.objects[o].state.q) - q).max() <= 1e-6 * np.abs(q).max()
    q0 = _h(sim.objects[0].state.q).reshape(-1, 3)
    assert np.array_equal(q0[g["fixed"]], g["lower_nodes"][g["fixed"]])
