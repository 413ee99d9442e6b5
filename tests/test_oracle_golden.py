"""Pin the CPU oracle (oracle/cn_oracle.py) to golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import cn_oracle as orc


def test_rebuild_violation_dt_bitwise(golden):
    g = golden("kat_rebuild.npz")
    for k in range(3):
        W = orc.rebuild_w(g[f"D{k}"], g[f"wg{k}"])
        assert np.array_equal(W, g[f"W{k}"])
        assert np.array_equal(orc.violation(g[f"D{k}"], g[f"pa{k}"], g[f"pb{k}"]), g[f"delta{k}"])
        assert np.array_equal(orc.apply_dt(g[f"D{k}"], g[f"lam{k}"]), g[f"dt{k}"])
    assert np.array_equal(orc.naive_gemm(g["gA"], g["gB"].T), g["gC"])


def test_pgs_matches_reference(golden):
    g = golden("kat_pgs.npz")
    for k in range(int(g["n"])):
        mu, tol, it = g[f"cfg{k}"]
        lam, dend, iters, eps, conv = orc.pgs(g[f"W{k}"], g[f"delta{k}"], 0.01, int(it), tol, mu)
        assert iters == int(g[f"it{k}"])
        assert conv == bool(g[f"conv{k}"])
        assert np.array_equal(lam, g[f"lam{k}"])
        assert np.array_equal(dend, g[f"dend{k}"])
        assert np.array_equal(np.array(eps), g[f"eps{k}"])


def test_frames_and_relinearize(golden):
    g = golden("kat_frames.npz")
    F = orc.detection_frames(g["p_a"], g["p_b"], g["ref"])
    assert np.array_equal(F, g["frames"])
    F2, rot = orc.relinearize(g["p_a2"], g["p_b"], F)
    assert np.array_equal(F2, g["frames2"])
    assert rot == float(g["rotation"])


def test_linear_system_and_factor(golden):
    g = golden("kat_linalg.npz")
    body = orc.Body(g["nodes"], g["tets"], young=5e4, poisson=0.3, fixed_nodes=[0, 1, 2])
    assert np.array_equal(body.masses, g["masses"])
    K = body.K
    assert np.array_equal(K.indptr, g["K_indptr"]) and np.array_equal(K.indices, g["K_indices"])
    assert np.abs(K.data - g["K_data"]).max() <= 1e-12 * np.abs(g["K_data"]).max()
    A, b = body.system(g["q"], g["v"], 0.01, (0.0, -9.81, 0.0))
    assert np.array_equal(A.indptr, g["indptr"]) and np.array_equal(A.indices, g["indices"])
    assert np.abs(A.data - g["data"]).max() <= 1e-12 * np.abs(g["data"]).max()
    assert np.abs(b - g["b"]).max() <= 1e-12 * np.abs(g["b"]).max()
    F = orc.Factor(A)
    assert np.abs(F.solve(g["b"]) - g["x"]).max() <= 1e-12 * np.abs(g["x"]).max()
    assert np.abs(F.solve(g["B"]) - g["X"]).max() <= 1e-12 * np.abs(g["X"]).max()


def _scene_from_fixture(g, n_obj, normal=(0.0, 1.0, 0.0), **kw):
    bodies = []
    vel = []
    for o in range(n_obj):
        E, nu, rho, a, b = g[f"mat{o}"]
        bodies.append(orc.Body(g[f"mesh{o}_nodes"], g[f"mesh{o}_tets"], young=E, poisson=nu,
                               density=rho, alpha=a, beta=b))
        vel.append(tuple(g[f"vel{o}"]))
    return orc.Scene(bodies, [dict(normal=np.array(normal), offset=0.0)], velocities=vel, **kw)


def _check_steps(sc, g, steps, rtol_q=1e-9):
    for s in range(steps):
        out = sc.step()
        assert out["n_pairs"] == int(g[f"s{s}_npairs"])
        if f"s{s}_keys" in g:
            keys = np.column_stack([out["pairs"][k] for k in ("obj_a", "obj_b", "vertex_id", "element_id")]) \
                if out["n_pairs"] else np.zeros((0, 4), dtype=np.int64)
            assert np.array_equal(keys.astype(np.int64), g[f"s{s}_keys"])
            if out["n_pairs"]:
                assert np.array_equal(out["frames"], g[f"s{s}_frames"])
                wg = g[f"s{s}_wg"]
                assert np.abs(out["wg"] - wg).max() <= 1e-12 * np.abs(wg).max()
                lh = np.stack(out["result"]["lam_history"])
                ref = g[f"s{s}_lamhist"]
                assert np.abs(lh - ref).max() <= 1e-9 * max(np.abs(ref).max(), 1e-300)
        for o in range(len(sc.bodies)):
            q = g[f"s{s}_q{o}"]
            assert np.abs(sc.q[o] - q).max() <= rtol_q * np.abs(q).max()


def test_block_on_plane_scene(golden):
    g = golden("block_on_plane.npz")
    sc = _scene_from_fixture(g, 1, threshold=0.01, mu=0.5, pgs_iter=300, pgs_tol=1e-10, newton_iter=4,
                             penetration_tol=-1.0, rotation_tol=-1.0)
    _check_steps(sc, g, 3)


def test_two_body_press_scene(golden):
    g = golden("two_body_press.npz")
    sc = _scene_from_fixture(g, 2, threshold=0.01, mu=0.5, pgs_iter=300, pgs_tol=1e-10, newton_iter=4,
                             penetration_tol=-1.0, rotation_tol=-1.0)
    _check_steps(sc, g, 2)


def test_beam_cfg0_scene(golden):
    g = golden("beam_cfg0.npz")
    body = orc.Body(g["nodes"], g["tets"], young=5e3, poisson=0.45, density=1000.0)
    sc = orc.Scene([body], [dict(normal=g["normal"], offset=0.0)], threshold=0.005, mu=0.5,
                   pgs_iter=1000, pgs_tol=1e-10, newton_iter=5, penetration_tol=-1.0, rotation_tol=-1.0)
    rng = np.random.default_rng(0)
    sc.q[0] = sc.q[0] + rng.uniform(-1e-4, 1e-4, sc.q[0].shape)
    _check_steps(sc, g, 6)
