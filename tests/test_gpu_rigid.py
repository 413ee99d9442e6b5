"""Rigid spheres: 6-DoF bodies (reference dynamics.py:214-249),
sphere-plane pairs with RIGID_LOCAL attachments (collision.py:290-316, mapping
rows [I, -skew(lever)] at 448-457), the rotation folded in at commit
(scene.py:452-460) — against a 14-step reference run of two spheres (one
spinning, anisotropic inertia) and a soft box on a 15-degree plane
(tests/golden/rigid_spheres.npz): pair keys and Newton iterations every step,
lambda history, q / v of every body and the spheres' rotations within 1e-6."""

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


def test_rigid_spheres_against_reference(cn, golden):
    g = golden("rigid_spheres.npz")
    box = cn.TetMesh(g["box_nodes"], g["box_tets"])
    objs = [cn.SoftSpec(name="box", mesh=box, young=2e4, poisson=0.3, density=800.0),
            cn.RigidSphereSpec(name="ball", mass=0.3, radius=0.02, position=(0.0, 0.0215, 0.0),
                               velocity=(0.2, -0.3, 0.0, 0.0, 0.0, 4.0), inertia=np.diag([1e-4, 1.2e-4, 0.8e-4])),
            cn.RigidSphereSpec(name="marble", mass=0.05, radius=0.01, position=(-0.06, 0.012, 0.03)),
            cn.PlaneSpec(name="ground", normal=tuple(g["normal"]), offset=0.0)]
    cfg = cn.SceneConfig(objects=objs, h=0.01, threshold=0.006,
                         pgs=cn.PgsConfig(max_iterations=500, tolerance=1e-11, friction=0.4),
                         newton=cn.NewtonConfig(scheme="fast", max_iterations=3, penetration_tol=-1.0,
                                                rotation_tol=-1.0),
                         output=cn.OutputConfig(snapshots=False, metrics=False))
    sim = cn.Simulation(cfg)
    assert sim.total_dofs() == 3 * len(g["box_nodes"]) + 12
    for s in range(14):
        rep = sim.step()
        assert rep.c_groups == int(g[f"s{s}_npairs"]), s
        assert rep.newton_iterations == int(g[f"s{s}_newton"])
        keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in sim.last_pairs]).reshape(-1, 4)
        assert np.array_equal(keys, g[f"s{s}_keys"]), s
        if f"s{s}_lamhist" in g:
            lh = _h(torch.stack(sim.last_result.lam_history))
            ref = g[f"s{s}_lamhist"]
            assert np.abs(lh - ref).max() <= 1e-6 * np.abs(ref).max(), s
        for obj in sim.dynamic_objects:
            q, v = g[f"s{s}_q{obj.oid}"], g[f"s{s}_v{obj.oid}"]
            assert np.abs(_h(obj.state.q) - q).max() <= 1e-6 * max(np.abs(q).max(), 1e-3), (s, obj.oid)
            assert np.abs(_h(obj.state.v) - v).max() <= 1e-6 * max(np.abs(v).max(), 1e-3), (s, obj.oid)
            if obj.kind == "rigid":
                assert np.abs(obj.rotation - g[f"s{s}_R{obj.oid}"]).max() <= 1e-9, (s, obj.oid)

