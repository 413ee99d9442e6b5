"""The benched corotational material against its CPU oracle (oracle/cn_oracle.py
``CorotBody``, pinned by tests/test_oracle_corot_cpu.py).

cnb_fe_element's rotations R_e, rotated blocks R K_e R^T and element forces
R K_e (R^T x - x0) at random deformed, near-degenerate and inverted states;
the assembled K(q), A and b (fixed DoFs included); and a 3-step two-block
corotational trajectory (per-step refactorisation) against the oracle scene."""

import numpy as np
import pytest
import torch
from scipy.spatial.transform import Rotation

import cn_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_06946_b200 as m

    return m


def _h(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _states(mesh, seed):
    rng = np.random.default_rng(seed)
    out = {}
    rot = Rotation.from_rotvec(rng.normal(size=3)).as_matrix()
    x = mesh.nodes @ rot.T + rng.normal(size=3) * 0.01
    out["deformed"] = (x + rng.uniform(-2e-3, 2e-3, x.shape)).ravel()
    # near-degenerate: squash y to 5 % and shear
    sq = mesh.nodes * np.array([1.0, 0.05, 1.0]) + np.outer(mesh.nodes[:, 1], [0.3, 0.0, 0.0])
    out["squashed"] = (sq @ rot.T).ravel()
    # inverted elements: a column of nodes pushed through the body
    inv = mesh.nodes.copy()
    top = mesh.nodes[:, 1] >= mesh.nodes[:, 1].max() - 1e-12
    inv[top, 1] -= 0.025
    out["inverted"] = (inv + rng.uniform(-1e-4, 1e-4, inv.shape)).ravel()
    return out


@pytest.mark.parametrize("which", ["deformed", "squashed", "inverted"])
def test_element_kernel_against_oracle(cn, which):
    mesh = cn.five_tet_grid((5, 3, 4), 0.01)
    body = cn.SoftBody(mesh, young=2e3, poisson=0.4, material="corotational")
    ob = orc.CorotBody(mesh.nodes, mesh.tets, young=2e3, poisson=0.4)
    q = _states(mesh, 7)[which]
    D = body._device()
    body._assemble_elements(torch.as_tensor(q, device="cuda"))
    R_o, Kb_o, fe_o, _ = ob.element_state(q)
    det = np.linalg.det(np.einsum("eai,eaj->eij", q.reshape(-1, 3)[mesh.tets], ob.grads))
    if which == "inverted":
        assert (det <= 0).any()
    R = _h(D["R"]).reshape(-1, 3, 3)
    Kb = _h(D["Kb"]).reshape(-1, 4, 4, 3, 3)
    fe = _h(D["fe"]).reshape(-1, 4, 3)
    # det F > 0: Newton polar iteration vs the SVD polar factor; det F <= 0:
    # Horn's quaternion eigenvector vs the SVD maximiser of tr(R^T F)
    tol = np.where(det > 1e-12, 1e-12, 1e-11)
    errR = np.abs(R - R_o).max(axis=(1, 2))
    assert np.all(errR <= tol), (errR.max(), which)
    kscale = np.abs(Kb_o).max()
    rel = 1e-11 if which == "inverted" else 1e-12
    assert np.abs(Kb - Kb_o).max() <= rel * kscale
    fscale = np.abs(fe_o).max()
    assert np.abs(fe - fe_o).max() <= rel * fscale


def test_assembled_system_against_oracle(cn):
    mesh = cn.five_tet_grid((6, 4, 4), 0.01, (0.0, 0.01, 0.0))
    fixed = np.array([0, 1, 2, 5, 9])
    body = cn.SoftBody(mesh, young=1e4, poisson=0.4, fixed_nodes=fixed, material="corotational")
    ob = orc.CorotBody(mesh.nodes, mesh.tets, young=1e4, poisson=0.4, fixed_nodes=fixed)
    q = _states(mesh, 3)["deformed"]
    v = np.random.default_rng(4).normal(size=q.shape) * 0.05
    A, b = body.assemble(cn.MechanicalState(q, v), 0.01, (0.0, -9.81, 0.0))
    Ao, bo = ob.system(q, v, 0.01, (0.0, -9.81, 0.0))
    csr = A.csr
    assert np.array_equal(csr.indptr, Ao.indptr) and np.array_equal(csr.indices, Ao.indices)
    assert np.abs(csr.data - Ao.data).max() <= 1e-12 * np.abs(Ao.data).max()
    assert np.abs(_h(b) - bo).max() <= 1e-12 * np.abs(bo).max()
    K = body.stiffness()
    Ko = ob.stiffness_at(q)
    assert np.abs((K - Ko).toarray()).max() <= 1e-12 * np.abs(Ko.data).max()
    f = _h(body.internal_force(q, v))
    fo = ob.internal_force(q, v)
    assert np.abs(f - fo).max() <= 1e-12 * np.abs(fo).max()


def test_two_block_corotational_trajectory(cn):
    """Upper block sliding over a lower block on the ground (the cfg3 setup at
    small size), corotational material, refactorised every step."""
    lower = cn.five_tet_grid((6, 3, 5), 0.01, (0.0, 0.0015, 0.0))
    upper = cn.five_tet_grid((4, 3, 4), 0.01, (0.01, 0.0225, 0.005))
    mats = [dict(young=1e4, poisson=0.4), dict(young=2e3, poisson=0.4)]
    vel = [(0.0, 0.0, 0.0), (0.5, 0.0, 0.0)]
    objs = [cn.SoftSpec(name=f"b{k}", mesh=m, density=1000.0, velocity=vel[k], material="corotational", **mats[k])
            for k, m in enumerate((lower, upper))]
    objs.append(cn.PlaneSpec(name="ground", normal=(0.0, 1.0, 0.0), offset=0.0))
    cfg = cn.SceneConfig(objects=objs, h=0.01, threshold=0.004,
                         pgs=cn.PgsConfig(max_iterations=300, tolerance=1e-10, friction=0.4),
                         newton=cn.NewtonConfig(scheme="fast", max_iterations=3, penetration_tol=-1.0,
                                                rotation_tol=-1.0),
                         output=cn.OutputConfig(snapshots=False, metrics=False))
    sim = cn.Simulation(cfg)
    bodies = [orc.CorotBody(m.nodes, m.tets, density=1000.0, **mats[k]) for k, m in enumerate((lower, upper))]
    osc = orc.Scene(bodies, [dict(normal=(0.0, 1.0, 0.0), offset=0.0)], h=0.01, threshold=0.004, mu=0.4,
                    pgs_iter=300, pgs_tol=1e-10, newton_iter=3, penetration_tol=-1.0, rotation_tol=-1.0,
                    velocities=vel)
    for s in range(3):
        rep = sim.step()
        out = osc.step()
        assert rep.c_groups == out["n_pairs"]
        keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in sim.last_pairs])
        okeys = np.stack([out["pairs"][k] for k in ("obj_a", "obj_b", "vertex_id", "element_id")], axis=1)
        assert np.array_equal(keys, okeys)
        lh = _h(torch.stack(sim.last_result.lam_history))
        ref = np.stack(out["result"]["lam_history"])
        assert np.abs(lh - ref).max() <= 1e-6 * np.abs(ref).max()
        for k in range(2):
            q = osc.q[k]
            assert np.abs(_h(sim.objects[k].state.q) - q).max() <= 1e-6 * np.abs(q).max(), (s, k)
