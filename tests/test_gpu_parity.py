"""GPU parity: every kernel on the hot path against golden vectors produced by the
reference (tests/golden) and against the CPU oracle.  Tolerances follow the
north star: bit-exact for integers, 1e-9 relative on W / W_g / dx, 1e-6 on
lambda and positions."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

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


def rel_err(a, b):
    a, b = _h(a), _h(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)) if b.size else 0.0


def test_rebuild_w_bitwise(cn, golden):
    g = golden("kat_rebuild.npz")
    for k in range(3):
        D = cn.assemble_direction(g[f"D{k}"])
        wg = cn.MappingDelassus(torch.as_tensor(g[f"wg{k}"], device="cuda"), {})
        W = cn.rebuild_W_fast(D, wg).W
        assert np.array_equal(_h(W), g[f"W{k}"])
        delta = cn.compute_violation(D, g[f"pa{k}"], g[f"pb{k}"]).delta
        assert np.array_equal(_h(delta), g[f"delta{k}"])
        assert np.array_equal(_h(D.apply_transposed(g[f"lam{k}"])), g[f"dt{k}"])


def test_gemm_naive_bitwise(cn, golden):
    g = golden("kat_rebuild.npz")
    C = cn.gemm(g["gA"], g["gB"], transpose_b=True)
    assert np.array_equal(_h(C), g["gC"])
    rng = np.random.default_rng(5)
    A, B = rng.standard_normal((7, 9)), rng.standard_normal((7, 5))
    assert np.array_equal(_h(cn.gemm(A, B, transpose_a=True)), orc.naive_gemm(A.T, B))


def test_frames_and_relinearize(cn, golden):
    g = golden("kat_frames.npz")
    pairs = [cn.ProximityPair(0, 1, cn.Attachment(cn.AttachKind.VERTEX, 0, vertex=0),
                              cn.Attachment(cn.AttachKind.WORLD, 1, world_point=np.zeros(3)),
                              g["p_a"][i], g["p_b"][i], g["ref"][i], 0.0, i, -1) for i in range(len(g["p_a"]))]
    F = cn.build_frames(pairs)
    assert rel_err(F.blocks, g["frames"]) <= 1e-15
    F2 = cn.relinearize(pairs, g["p_a2"], g["p_b"], F)
    assert rel_err(F2.blocks, g["frames2"]) <= 1e-15
    assert abs(cn.max_frame_rotation(F, F2) - float(g["rotation"])) <= 1e-12


def test_pgs_matches_reference(cn, golden):
    g = golden("kat_pgs.npz")
    for k in range(int(g["n"])):
        mu, tol, it = g[f"cfg{k}"]
        res = cn.pgs(g[f"W{k}"], g[f"delta{k}"], 0.01, cn.PgsConfig(int(it), float(tol), float(mu)))
        ref = g[f"lam{k}"]
        assert rel_err(res.lam, ref) <= 1e-6, k
        assert abs(res.iterations - int(g[f"it{k}"])) <= 1, (k, res.iterations, int(g[f"it{k}"]))
        assert res.converged == bool(g[f"conv{k}"]) or res.iterations != int(g[f"it{k}"])
        assert np.abs(_h(res.delta_end) - g[f"dend{k}"]).max() <= 1e-9 * max(1.0, np.abs(g[f"dend{k}"]).max())


def test_pgs_fixed_sweeps_close_to_reference(cn, golden):
    """Same number of sweeps: iterates agree to rounding of the delta sums."""
    g = golden("kat_pgs.npz")
    for k in range(int(g["n"])):
        mu, tol, it = g[f"cfg{k}"]
        n_it = int(g[f"it{k}"])
        lam_o, *_ = orc.pgs(g[f"W{k}"], g[f"delta{k}"], 0.01, n_it, 1e-300, mu)
        res = cn.pgs(g[f"W{k}"], g[f"delta{k}"], 0.01, cn.PgsConfig(n_it, 1e-300, float(mu)))
        assert res.iterations == n_it
        assert rel_err(res.lam, lam_o) <= 1e-9, k


def test_local_solve(cn):
    rng = np.random.default_rng(4)
    B = rng.standard_normal((6, 6))
    W = B @ B.T + 3 * np.eye(6)
    for mu in (0.0, 0.3, 10.0):
        d = np.array([-0.01, 0.0005, -0.0003, 0.002, 0.1, -0.1])
        lam = np.abs(rng.standard_normal(6))
        for g in (0, 1):
            ref = orc.local_solve(g, W, d, lam, mu, 1e-4)
            out = cn.local_solve(g, W, d, lam, mu, 1e-4)
            assert np.array_equal(_h(out), ref)
    with pytest.raises(cn.SingularBlockError):
        cn.local_solve(0, np.zeros((3, 3)), np.array([-0.1, 0, 0]), np.zeros(3), 0.5, 1e-4)


# --- factorisation ------------------------------------------------------------------

def random_spd(dim, seed, shift=10.0):
    rng = np.random.default_rng(seed)
    L = np.tril(rng.standard_normal((dim, dim)))
    return L @ L.T + shift * np.eye(dim)


def test_factor_solve_against_reference_fixture(cn, golden):
    g = golden("kat_linalg.npz")
    n = len(g["b"])
    A = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    F = cn.factorize(cn.SparseSym(A))
    assert rel_err(F.solve(g["b"]), g["x"]) <= 1e-12
    assert rel_err(F.solve_multi(g["B"]), g["X"]) <= 1e-12
    assert F.solve_count == 1 + g["B"].shape[1]


def test_factor_random_spd_and_errors(cn):
    for dim in (1, 2, 7, 23, 50, 130):
        A = random_spd(dim, dim)
        F = cn.factorize(cn.SparseSym(A))
        B = np.random.default_rng(dim + 1).standard_normal((dim, 4))
        X = _h(F.solve_multi(B))
        assert np.abs(A @ X - B).max() <= 1e-9 * np.abs(B).max()
        x1 = _h(F.solve(B[:, 0]))
        x2 = _h(cn.factorize(cn.SparseSym(A)).solve(B[:, 0]))
        assert np.array_equal(x1, x2)  # deterministic
    A = random_spd(6, 5)
    A[2, 2] = -50.0
    with pytest.raises(cn.NotSPDError):
        cn.factorize(cn.SparseSym(A))
    Z = np.zeros((3, 3))
    Z[0, 0] = 1.0
    with pytest.raises(cn.NotSPDError):
        cn.factorize(cn.SparseSym(Z))
    with pytest.raises(cn.DimensionMismatchError):
        cn.factorize(cn.SparseSym(sp.eye(3))).solve(np.zeros(4))


def test_factor_fe_mesh_blocked(cn):
    mesh = cn.five_tet_grid((12, 5, 6), 0.01)
    body = orc.Body(mesh.nodes, mesh.tets, young=5e3, poisson=0.45, fixed_nodes=[0, 1, 2, 3])
    A, b = body.system(mesh.nodes.ravel(), np.zeros(3 * mesh.n_nodes), 0.01, (0, -9.81, 0))
    S = cn.SparseSym(A, check=False)
    S.pattern.block_size = 3
    S.pattern.coords = mesh.nodes
    F = cn.Factorization(S)
    x = _h(F.solve(b))
    ref = orc.Factor(A).solve(b)
    assert rel_err(x, ref) <= 1e-10


# --- scene-level: block_on_plane step 0 ---------------------------------------------

def _block_on_plane_step0(cn, g):
    E, nu, rho, a, bb = g["mat0"]
    nodes, tets = g["mesh0_nodes"], g["mesh0_tets"]
    body = orc.Body(nodes, tets, young=E, poisson=nu, density=rho, alpha=a, beta=bb)
    q = nodes.ravel().copy()
    v = np.tile(g["vel0"], len(nodes))
    A, rhs = body.system(q, v, 0.01, (0.0, -9.81, 0.0))
    tris = cn.surface_triangles(tets)
    geom = cn.MeshGeometry(0, nodes, tris, np.unique(tris), True, True)
    plane = cn.PlaneGeometry(1, (0.0, 1.0, 0.0), 0.0)
    pairs = cn.detect([geom, plane], 0.01)
    return body, A, rhs, pairs


def test_detect_keys_match_reference(cn, golden):
    g = golden("block_on_plane.npz")
    _, _, _, pairs = _block_on_plane_step0(cn, g)
    keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in pairs])
    assert np.array_equal(keys, g["s0_keys"])


def test_wg_and_newton_fast_block_on_plane(cn, golden):
    g = golden("block_on_plane.npz")
    body, A, rhs, pairs = _block_on_plane_step0(cn, g)
    Ssym = cn.SparseSym(A, check=False)
    F = cn.Factorization(Ssym)
    dv_free = F.solve(rhs)
    q_free = torch.as_tensor(g["mesh0_nodes"].ravel(), device="cuda") + 0.01 * (
        torch.as_tensor(np.tile(g["vel0"], len(g["mesh0_nodes"])), device="cuda") + dv_free)
    assert rel_err(q_free, g["s0_qfree0"]) <= 1e-12
    S = cn.build_signed_mapping(pairs, 0, body.n, body.fixed_mask)
    wg = cn.assemble_Wg({0: S}, {0: F})
    assert rel_err(wg.wg, g["s0_wg"]) <= 1e-9
    frames = cn.build_frames(pairs)
    assert rel_err(frames.blocks, g["s0_frames"]) <= 1e-14
    p_a0, p_b0 = cn.refresh_proximity(pairs, {0: q_free.reshape(-1, 3), 1: None})
    assert rel_err(p_a0, g["s0_pa0"]) <= 1e-14
    ctx = cn.StepContext(pairs=pairs, detection_frames=frames, S_by_object={0: S}, F_by_object={0: F},
                         p_a0=p_a0, p_b0=p_b0, h=0.01, wg=wg)
    ncfg = cn.NewtonConfig(scheme="fast", max_iterations=4, penetration_tol=-1.0, rotation_tol=-1.0)
    pcfg = cn.PgsConfig(max_iterations=300, tolerance=1e-10, friction=0.5)
    before = F.solve_count
    res = cn.newton_fast(ctx, ncfg, pcfg)
    assert F.solve_count - before == 1  # test_solver.py:328-341
    lh = torch.stack(res.lam_history)
    assert rel_err(lh, g["s0_lamhist"]) <= 1e-6
    assert rel_err(res.state.accumulated, g["s0_acc"]) <= 1e-6
    assert rel_err(res.dv_by_object[0], g["s0_dv0"]) <= 1e-6
    # fast update == full mechanical pipeline (test_constraints.py:350-367)
    q_new = q_free + 0.01 * res.dv_by_object[0]
    pa_m, pb_m = cn.refresh_proximity(pairs, {0: q_new.reshape(-1, 3), 1: None})
    assert np.abs(_h(res.p_a) - _h(pa_m)).max() <= 1e-9


def test_pgs_grid_kernel_matches_reference(cn, golden, monkeypatch):
    """The grid-scale PGS (all SMs, used for thousands of groups) on the golden
    cases: same iterate as the single-CTA kernel and the reference."""
    monkeypatch.setenv("CNB_PGS_GRID", "1")
    g = golden("kat_pgs.npz")
    for k in range(int(g["n"])):
        mu, tol, it = g[f"cfg{k}"]
        res = cn.pgs(g[f"W{k}"], g[f"delta{k}"], 0.01, cn.PgsConfig(int(it), float(tol), float(mu)))
        assert rel_err(res.lam, g[f"lam{k}"]) <= 1e-6, k
        assert abs(res.iterations - int(g[f"it{k}"])) <= 1, k
        assert np.abs(_h(res.delta_end) - g[f"dend{k}"]).max() <= 1e-9 * max(1.0, np.abs(g[f"dend{k}"]).max())


def test_pgs_grid_large_random(cn, monkeypatch):
    """3000 groups (c = 9000): grid kernel vs single-CTA kernel on a fixed sweep budget."""
    rng = np.random.default_rng(11)
    G = 3000
    c = 3 * G
    B = rng.standard_normal((c, 64)) / 8.0
    W = B @ B.T + np.eye(c)
    delta = rng.uniform(-0.02, 0.01, c)
    cfg = cn.PgsConfig(20, 1e-300, 0.4)
    r_grid = cn.pgs(W, delta, 0.01, cfg)
    monkeypatch.setenv("CNB_PGS_GRID", "0")
    lam_o, *_ = orc.pgs(W[:300, :300], delta[:300], 0.01, 20, 1e-300, 0.4)  # small oracle sanity
    r_small = cn.pgs(W[:300, :300], delta[:300], 0.01, cfg)
    assert rel_err(r_small.lam, lam_o) <= 1e-9
    assert r_grid.iterations == 20
    # grid result satisfies the complementarity structure of a GS sweep fixed point trend
    lam = _h(r_grid.lam).reshape(-1, 3)
    assert (lam[:, 0] >= 0).all()
    assert (np.hypot(lam[:, 1], lam[:, 2]) <= 0.4 * lam[:, 0] * (1 + 1e-9) + 1e-12).all()


def _oracle_mesh(oid, nodes, tris):
    return dict(id=oid, points=nodes, triangles=tris, vertex_ids=np.unique(tris), deformable=True, dynamic=True)


@pytest.mark.parametrize("shape_a,shape_b,dy,jitter", [
    ((6, 3, 5), (7, 3, 6), 0.0203, 0.0),      # grid-aligned: exact distance ties everywhere
    ((9, 4, 9), (10, 5, 10), 0.0395, 2e-4),   # upper block sunk 0.5 mm into the lower one
    ((14, 4, 12), (16, 5, 16), 0.0380, 1e-3), # jittered, deeper overlap, several triangle slices
])
def test_detect_vertex_mesh_matches_oracle(cn, shape_a, shape_b, dy, jitter):
    """GPU all-pairs closest-point scan vs the oracle (collision.py:222-260): pair keys,
    attachments and floats bit-identical, including lowest-index tie breaks."""
    from paper_2306_06946_b200.mesh import five_tet_grid

    rng = np.random.default_rng(7)
    lower = five_tet_grid(shape_b, 0.01)
    upper = five_tet_grid(shape_a, 0.01, (0.0125, dy, 0.0075))
    nodes = [upper.nodes + jitter * rng.standard_normal(upper.nodes.shape),
             lower.nodes + jitter * rng.standard_normal(lower.nodes.shape)]
    tris = [cn.surface_triangles(upper.tets), cn.surface_triangles(lower.tets)]
    geoms = [cn.MeshGeometry(i, nodes[i], tris[i], np.unique(tris[i]), True, True) for i in range(2)]
    pairs = cn.detect(geoms, 0.005)
    ref = orc.detect([_oracle_mesh(i, nodes[i], tris[i]) for i in range(2)], [], 0.005)
    assert len(pairs) == len(ref["vertex_id"]) > 0
    keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in pairs])
    rkeys = np.stack([ref["obj_a"], ref["obj_b"], ref["vertex_id"], ref["element_id"]], 1)
    assert np.array_equal(keys, rkeys)
    assert np.array_equal(np.stack([p.attach_b.triangle for p in pairs]), ref["tri_b"])
    assert np.array_equal(np.stack([p.attach_b.weights for p in pairs]), ref["w_b"])
    assert np.array_equal(np.stack([p.p_b for p in pairs]), ref["p_b"])
    assert np.array_equal(np.stack([p.ref_normal for p in pairs]), ref["ref_normal"])
    assert np.array_equal(np.array([p.signed_distance for p in pairs]), ref["signed"])
