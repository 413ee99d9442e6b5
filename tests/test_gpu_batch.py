"""Batched independent scenes (BASELINE configs[4]) against the reference's
cfg0 trajectory (tests/golden/beam_cfg0.npz, made by the reference) and
against one ``Simulation`` per copy: same pair vertex sets (bit-exact), same
node positions within 1e-6 relative (north_star tolerance)."""

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
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_batched_copies_follow_reference_cfg0(cn, golden):
    """Copies 0 and 2 are the golden cfg0 run; copy 1 (other tilt / mu) sits between
    them and must not disturb them."""
    from paper_2306_06946_b200.batch import BatchedPlaneScenes, placement, plane_normals

    g = golden("beam_cfg0.npz")
    nodes, tets = g["nodes"], g["tets"]
    mesh = cn.TetMesh(nodes, tets)
    n = nodes.size
    tilts = [10.0, 17.0, 10.0]
    rest = np.stack([nodes, placement(nodes, plane_normals([17.0]), 0.002)[0], nodes])
    jit0 = np.random.default_rng(0).uniform(-1e-4, 1e-4, n)
    jitter = np.stack([jit0, np.random.default_rng(7).uniform(-1e-4, 1e-4, n), jit0])
    normals = np.stack([g["normal"], plane_normals([17.0])[0], g["normal"]])
    B = BatchedPlaneScenes(mesh, tilts, [0.5, 0.3, 0.5], jitter, threshold=0.005, rest_nodes=rest, normals=normals)
    # the normals are the golden's to the bit
    assert np.array_equal(_h(B.normals[0]), g["normal"])
    for s in range(6):
        B.step()
        B.check()
        P = B.last["pairs"] if B.last else None
        for c in (0, 2):
            cnt = int(P["cnt"][c]) if P is not None else 0
            assert cnt == int(g[f"s{s}_npairs"]), (s, c)
            if f"s{s}_keys" in g and cnt:
                assert np.array_equal(B.pair_keys(c), g[f"s{s}_keys"][:, 2])
            q = g[f"s{s}_q0"]
            assert _rel(_h(B.Q[c]), q) <= 1e-6, (s, c, _rel(_h(B.Q[c]), q))
        assert np.array_equal(_h(B.Q[0]), _h(B.Q[2]))  # copies are independent and deterministic


def test_batched_copies_match_simulation(cn):
    """cfg4 draws for three copies vs one Simulation.step per copy."""
    from paper_2306_06946_b200.batch import BatchedPlaneScenes, cfg4_draws, placement, plane_normals

    mesh = cn.five_tet_grid((20, 4, 4), 0.01)
    n = mesh.nodes.size
    tilts, mus, jit = cfg4_draws(0, 3, n)
    B = BatchedPlaneScenes(mesh, tilts, mus, jit, threshold=0.005, clearance=0.002)
    rest = placement(mesh.nodes, plane_normals(tilts), 0.002)
    sims = []
    for i in range(3):
        cfg = cn.SceneConfig(
            objects=[cn.SoftSpec(name="beam", mesh=cn.TetMesh(rest[i], mesh.tets), young=5e3, poisson=0.45,
                                 density=1000.0),
                     cn.PlaneSpec(name="ground", normal=tuple(plane_normals([tilts[i]])[0]), offset=0.0)],
            threshold=0.005, pgs=cn.PgsConfig(1000, 1e-10, float(mus[i])),
            newton=cn.NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0, rotation_tol=-1.0),
            output=cn.OutputConfig(snapshots=False, metrics=False))
        sim = cn.Simulation(cfg)
        st = sim.objects[0].state
        sim.objects[0].state = cn.MechanicalState(_h(st.q) + jit[i], st.v)
        sims.append(sim)
    lam_scale = 0.01 * 9.81 * float(B.body.masses().sum())
    seen = 0
    for s in range(6):
        B.step()
        B.check()
        for i, sim in enumerate(sims):
            rep = sim.step()
            cnt = int(B.last["pairs"]["cnt"][i]) if B.last else 0
            assert cnt == rep.c_groups, (s, i)
            if cnt:
                seen += 1
                ref = np.array([p.vertex_id for p in sim.last_pairs])
                assert np.array_equal(B.pair_keys(i), ref)
                lam_ref = _h(sim.last_lam)
                P = B.last["pairs"]
                a, b = 3 * int(P["poff_h"][i]), 3 * int(P["poff_h"][i + 1])
                err = np.abs(_h(B.last["lam"][a:b]) - lam_ref).max()
                # floor: one step's weight impulse (resting contacts carry round-off-sized lambdas)
                assert err <= 1e-6 * max(np.abs(lam_ref).max(), lam_scale), (s, i, err)
            q = _h(sim.objects[0].state.q)
            assert _rel(_h(B.Q[i]), q) <= 1e-6, (s, i, _rel(_h(B.Q[i]), q))
            v = _h(sim.objects[0].state.v)
            assert np.abs(_h(B.V[i]) - v).max() <= 1e-6 * max(np.abs(v).max(), 1e-3)
    assert seen >= 6  # contacts were exercised


def test_batched_no_contacts_is_free_fall(cn):
    """Copies far above their planes: no pairs, q follows the free motion of a
    single Simulation exactly (same factor, same right-hand side)."""
    from paper_2306_06946_b200.batch import BatchedPlaneScenes

    mesh = cn.five_tet_grid((6, 3, 3), 0.01)
    B = BatchedPlaneScenes(mesh, [0.0, 5.0], [0.5, 0.5], None, clearance=0.5)
    for _ in range(3):
        assert B.step() == 0
    B.check()
    assert np.isfinite(_h(B.Q)).all()
    # both copies fall by the same amount along y, the motion is a pure translation
    d = _h(B.Q) - B.rest_host
    assert np.abs(d[0] - d[1]).max() <= 1e-12
    assert (d.reshape(2, -1, 3)[:, :, 1] < 0).all()


def test_plane_distances_bit_exact(cn):
    """Device plane distances equal the reference's per-vertex float(n @ p - offset)
    bit for bit (numpy's 3-element dot is a fused multiply-add chain)."""
    from paper_2306_06946_b200 import _device as dv
    from paper_2306_06946_b200 import _lib

    rng = np.random.default_rng(11)
    pts = rng.uniform(-0.3, 0.3, (5000, 3))
    vids = np.sort(rng.choice(5000, 3000, replace=False)).astype(np.int64)
    for _ in range(3):
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        off = float(rng.uniform(-0.01, 0.01))
        out = dv.empty(len(vids))
        d_vids, d_pts = dv.upload(vids), dv.f64(pts)  # keep the device copies alive across the launch
        _lib.call("cnb_plane_distances", len(vids), d_vids.data_ptr(), d_pts.data_ptr(), float(n[0]),
                  float(n[1]), float(n[2]), off, out.data_ptr(), _lib.stream())
        ref = np.array([float(n @ pts[v] - off) for v in vids])
        assert np.array_equal(_h(out), ref)
