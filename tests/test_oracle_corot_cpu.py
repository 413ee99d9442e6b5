"""Pins of the corotational CPU oracle (oracle/cn_oracle.py ``CorotBody``).

The reference has no corotational material, so the oracle
that checks the benched material is pinned by its own defining properties:
  * at rest it IS the reference's linear material (K, A, b identical to the
    linear restatement, which tests/test_oracle_golden.py pins to the
    reference's own fixtures);
  * under a rigid motion the elastic force vanishes and K is rotated;
  * K(q) is symmetric;
  * f_el equals the gradient of the element energy 1/2 sum u^T K_e u
    (central finite differences) at a strongly deformed state.
"""

import numpy as np
import pytest
from scipy.linalg import polar
from scipy.spatial.transform import Rotation

import cn_oracle as orc
from paper_2306_06946_b200.mesh import five_tet_grid


@pytest.fixture(scope="module")
def block():
    mesh = five_tet_grid((4, 3, 3), 0.01, (0.0, 0.01, 0.0))
    return mesh, orc.CorotBody(mesh.nodes, mesh.tets, young=5e3, poisson=0.45, fixed_nodes=[0, 1])


def _deformed(mesh, seed, amp=2e-3):
    rng = np.random.default_rng(seed)
    rot = Rotation.from_rotvec(rng.normal(size=3) * 0.6).as_matrix()
    x = mesh.nodes @ rot.T + rng.normal(size=3) * 0.01
    return (x + rng.uniform(-amp, amp, x.shape)).ravel()


def test_rest_state_is_the_linear_material(block):
    mesh, cb = block
    lin = orc.Body(mesh.nodes, mesh.tets, young=5e3, poisson=0.45, fixed_nodes=[0, 1])
    q = mesh.nodes.ravel().copy()
    v = np.random.default_rng(0).normal(size=q.shape) * 0.01
    assert np.abs(cb.rotations(q) - np.eye(3)).max() <= 1e-14  # F = I up to the rounding of sum x_a g_a^T
    Kc, Kl = cb.stiffness_at(q), lin.K
    assert np.array_equal(Kc.indptr, Kl.indptr) and np.array_equal(Kc.indices, Kl.indices)
    assert np.abs(Kc.data - Kl.data).max() <= 1e-14 * np.abs(Kl.data).max()
    assert np.abs(cb.elastic_force(q)).max() <= 1e-14 * np.abs(Kl.data).max() * 1e-2
    Ac, bc = cb.system(q, v, 0.01, (0, -9.81, 0))
    Al, bl = lin.system(q, v, 0.01, (0, -9.81, 0))
    assert np.array_equal(Ac.indptr, Al.indptr) and np.array_equal(Ac.indices, Al.indices)
    assert np.abs(Ac.data - Al.data).max() <= 1e-14 * np.abs(Al.data).max()
    assert np.abs(bc - bl).max() <= 1e-12 * np.abs(bl).max()


def test_rigid_motion_zero_force_rotated_stiffness(block):
    mesh, cb = block
    Q = Rotation.from_rotvec([0.3, -1.1, 0.7]).as_matrix()
    x = mesh.nodes @ Q.T + np.array([0.05, -0.02, 0.01])
    q = x.ravel()
    R = cb.rotations(q)
    assert np.abs(R - Q).max() <= 1e-13
    scale = np.abs(cb.K.data).max() * 1e-2
    assert np.abs(cb.elastic_force(q)).max() <= 1e-11 * scale
    Kq = cb.stiffness_at(q).toarray()
    B = np.kron(np.eye(len(mesh.nodes)), Q)
    assert np.abs(Kq - B @ cb.K.toarray() @ B.T).max() <= 1e-12 * np.abs(cb.K.data).max()


def test_symmetric_and_polar_factor(block):
    mesh, cb = block
    q = _deformed(mesh, 1)
    K = cb.stiffness_at(q)
    assert abs(K - K.T).max() <= 1e-13 * np.abs(K.data).max()
    x = q.reshape(-1, 3)
    F = np.einsum("eai,eaj->eij", x[mesh.tets], cb.grads)
    R = cb.rotations(q)
    for e in range(0, len(mesh.tets), 7):
        u, _ = polar(F[e])
        assert np.abs(R[e] - u).max() <= 1e-13
    assert np.abs(np.einsum("eji,ejk->eik", R, R) - np.eye(3)).max() <= 1e-14
    assert np.all(np.linalg.det(R) > 0)


def test_force_is_energy_gradient(block):
    mesh, cb = block
    q = _deformed(mesh, 2, amp=3e-3)
    f = cb.elastic_force(q)
    rng = np.random.default_rng(3)
    eps = 1e-7
    for _ in range(6):
        d = rng.normal(size=q.shape)
        d /= np.linalg.norm(d)
        fd = (cb.energy(q + eps * d) - cb.energy(q - eps * d)) / (2 * eps)
        assert abs(fd - f @ d) <= 1e-6 * np.linalg.norm(f), (fd, f @ d)


def test_inverted_element_rotation_is_proper():
    F = np.diag([1.0, 0.8, -0.3])
    F = Rotation.from_rotvec([0.2, 0.4, -0.1]).as_matrix() @ F
    R = orc.rotation_factor(F[None])[0]
    assert abs(np.linalg.det(R) - 1.0) <= 1e-14
    # maximises tr(R^T F) over sampled rotations
    best = np.trace(R.T @ F)
    for rv in np.random.default_rng(4).normal(size=(200, 3)):
        assert np.trace(Rotation.from_rotvec(rv).as_matrix().T @ F) <= best + 1e-12
