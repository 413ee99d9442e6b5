"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The fixtures pin the oracle (oracle/cn_oracle.py)
and the CUDA path to the reference's own outputs; /root/reference is never
read at test time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import contactnewton as cn  # noqa: E402  (the reference)
from contactnewton import collision as rcol  # noqa: E402
from contactnewton import constraints as rcon  # noqa: E402
from contactnewton import scene as rsc  # noqa: E402
from contactnewton import solver as rsol  # noqa: E402

from paper_2306_06946_b200.mesh import five_tet_grid  # noqa: E402  (shared input generator)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def random_frame(rng):
    n = rng.standard_normal(3)
    n /= np.linalg.norm(n)
    t1 = np.cross(n, rng.standard_normal(3))
    t1 /= np.linalg.norm(t1)
    return rcol.ContactFrame(n=n, t1=t1, t2=np.cross(n, t1))


def kat_rebuild():
    rng = np.random.default_rng(100)
    out = {}
    for k, groups in enumerate((1, 7, 40)):
        c = 3 * groups
        B = rng.standard_normal((c, c))
        wg = B @ B.T / c + np.eye(c)
        frames = [random_frame(rng) for _ in range(groups)]
        D = rcon.assemble_direction(frames)
        W = rcon.rebuild_W_fast(D, rcon.MappingDelassus(wg, {0: wg})).W
        out[f"wg{k}"], out[f"D{k}"], out[f"W{k}"] = wg, D.blocks, W
        p_a, p_b = rng.standard_normal((groups, 3)), rng.standard_normal((groups, 3))
        out[f"pa{k}"], out[f"pb{k}"] = p_a, p_b
        out[f"delta{k}"] = rcon.compute_violation(D, p_a, p_b).delta
        lam = rng.standard_normal(c)
        out[f"lam{k}"], out[f"dt{k}"] = lam, D.apply_transposed(lam)
    A = rng.standard_normal((5, 4))
    Bm = rng.standard_normal((6, 4))
    out["gA"], out["gB"] = A, Bm
    out["gC"] = cn.gemm(A, Bm, transpose_b=True)
    save("kat_rebuild.npz", **out)


def kat_pgs():
    rng = np.random.default_rng(200)
    cases = []
    # (groups, mu, tol, max_iter, cond-ish)
    specs = [(1, 0.0, 1e-6, 30), (3, 0.4, 1e-6, 200), (5, 0.5, 1e-10, 1000), (33, 0.5, 1e-10, 500),
             (70, 0.3, 1e-8, 300), (70, 0.0, 1e-12, 2000), (100, 0.8, 1e-6, 30)]
    out = {}
    for k, (G, mu, tol, it) in enumerate(specs):
        c = 3 * G
        B = rng.standard_normal((c, c + 4))
        W = B @ B.T / c + 0.05 * np.eye(c)
        delta = rng.uniform(-0.02, 0.01, c)
        res = rsol.pgs(W, delta, 0.01, rsol.PgsConfig(max_iterations=it, tolerance=tol, friction=mu))
        out.update({f"W{k}": W, f"delta{k}": delta, f"lam{k}": res.lam, f"dend{k}": res.delta_end,
                    f"eps{k}": np.array(res.eps_history), f"it{k}": res.iterations,
                    f"conv{k}": res.converged, f"cfg{k}": np.array([mu, tol, it])})
    # duplicated contact -> regularisation path (test_solver.py:215-226 shape)
    W1 = np.eye(3)
    W = np.block([[W1, W1], [W1, W1]])
    delta = np.array([-0.01, 0, 0, -0.01, 0, 0.0])
    res = rsol.pgs(W, delta, 0.01, rsol.PgsConfig(max_iterations=300, tolerance=1e-10))
    k = len(specs)
    out.update({f"W{k}": W, f"delta{k}": delta, f"lam{k}": res.lam, f"dend{k}": res.delta_end,
                f"eps{k}": np.array(res.eps_history), f"it{k}": res.iterations,
                f"conv{k}": res.converged, f"cfg{k}": np.array([0.5, 1e-10, 300])})
    out["n"] = len(specs) + 1
    save("kat_pgs.npz", **out)


def kat_frames():
    rng = np.random.default_rng(300)
    m = 64
    p_b = rng.standard_normal((m, 3))
    d = rng.standard_normal((m, 3)) * 1e-3
    d[3] = 0.0  # coincident -> element normal fallback
    d[5] = np.array([0.0, 0.0, 1e-3])  # normal along z (tangent fallback axis)
    d[7] = np.array([1e-3, 0.0, 0.0])  # normal along x -> e_z fallback for t1
    ref = rng.standard_normal((m, 3))
    ref /= np.linalg.norm(ref, axis=1, keepdims=True)
    ref[7] = np.array([1.0, 0.0, 0.0])
    p_a = p_b + d
    pairs = [rcol.ProximityPair(0, 1, None, None, p_a[i], p_b[i], ref[i], 0.0, i, -1) for i in range(m)]
    frames = rcol.build_frames(pairs)
    F = np.stack([f.as_matrix() for f in frames])
    # relinearise: small motions, one collapse, one > 60 degree tilt
    p_a2 = p_a + rng.standard_normal((m, 3)) * 2e-4
    p_a2[10] = p_b[10]
    p_a2[11] = p_b[11] + 1e-3 * np.cross(F[11, 0], F[11, 1])  # 90 degrees away
    new = rcol.relinearize(pairs, p_a2, p_b, frames)
    rot = rcol.max_frame_rotation(frames, new)
    save("kat_frames.npz", p_a=p_a, p_b=p_b, ref=ref, frames=F, p_a2=p_a2,
         frames2=np.stack([f.as_matrix() for f in new]), rotation=rot)


def _run_scene(config, steps, capture_steps, jitter_seed=None, tag=""):
    sim = rsc.Simulation(config)
    if jitter_seed is not None:
        rng = np.random.default_rng(jitter_seed)
        for obj in sim.dynamic_objects:
            obj.state.q = obj.state.q + rng.uniform(-1e-4, 1e-4, obj.state.q.shape)
    out = {}
    for s in range(steps):
        if s in capture_steps:
            ctx, free, states, pen_before, timings, t_next = sim.prepare_step(build_wg=True)
            res = rsol.newton_fast(ctx, config.newton, config.pgs)
            keys = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in ctx.pairs],
                            dtype=np.int64).reshape(-1, 4)
            out[f"s{s}_keys"] = keys
            out[f"s{s}_frames"] = np.stack([f.as_matrix() for f in ctx.detection_frames]) if ctx.pairs \
                else np.zeros((0, 3, 3))
            out[f"s{s}_pa0"], out[f"s{s}_pb0"] = ctx.p_a0, ctx.p_b0
            if ctx.pairs:
                out[f"s{s}_wg"] = ctx.wg.wg
                for oid, U in ctx.wg.per_object.items():
                    out[f"s{s}_U{oid}"] = U
                out[f"s{s}_lamhist"] = np.stack(res.lam_history) if res.lam_history else np.zeros((0, 0))
                out[f"s{s}_acc"] = res.state.accumulated
                out[f"s{s}_final_frames"] = np.stack([f.as_matrix() for f in res.final_frames])
                for oid, dv in res.dv_by_object.items():
                    out[f"s{s}_dv{oid}"] = dv
                out[f"s{s}_sweeps"] = np.array([it.pgs_iterations for it in res.iterations])
                out[f"s{s}_rot"] = np.array([it.rotation for it in res.iterations])
            for obj in sim.dynamic_objects:
                out[f"s{s}_qfree{obj.oid}"] = free[obj.oid].q_free
            out[f"s{s}_pen_before"] = pen_before
        rep = sim.step()
        out[f"s{s}_npairs"] = rep.c_groups
        out[f"s{s}_newton"] = rep.newton_iterations
        out[f"s{s}_pen_after"] = rep.pen_after
        for obj in sim.dynamic_objects:
            out[f"s{s}_q{obj.oid}"] = obj.state.q.copy()
            out[f"s{s}_v{obj.oid}"] = obj.state.v.copy()
        print(tag, "step", s, "pairs", rep.c_groups, "newton", rep.newton_iterations,
              "pgs", rep.pgs_iterations_total, "pen_after", rep.pen_after)
    return out


def beam_cfg0(steps=10, drop=0.02):
    """BASELINE cfg0: 20x4x4-node 5-tet beam over a 10-degree plane."""
    ang = np.deg2rad(10.0)
    normal = np.array([np.sin(ang), np.cos(ang), 0.0])
    y0 = drop / normal[1]
    mesh = five_tet_grid((20, 4, 4), 0.01, (0.0, y0, 0.0))
    soft = rsc.SoftSpec(name="beam", mesh=cn.TetMesh(mesh.nodes, mesh.tets), young=5e3, poisson=0.45,
                        density=1000.0, rayleigh_mass=0.1, rayleigh_stiffness=0.1)
    plane = rsc.PlaneSpec(name="ground", normal=tuple(normal), offset=0.0)
    cfg = rsc.SceneConfig(objects=[soft, plane], h=0.01, threshold=0.005,
                          pgs=rsol.PgsConfig(max_iterations=1000, tolerance=1e-10, friction=0.5),
                          newton=rsol.NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1,
                                                   rotation_tol=-1),
                          output=rsc.OutputConfig(snapshots=False, metrics=False))
    return cfg, mesh


def scenes():
    # cfg0 beam, started 2 mm above the plane so contacts appear in step 1
    cfg, mesh = beam_cfg0(drop=0.002)
    out = _run_scene(cfg, 6, {2, 4}, jitter_seed=0, tag="beam")
    out.update(nodes=mesh.nodes, tets=mesh.tets, normal=np.array(cfg.objects[1].normal))
    save("beam_cfg0.npz", **out)
    # reference fixtures, forced fast scheme
    ref_scenes = "/root/reference/pkg/scenes"
    for name, steps, cap in (("block_on_plane", 3, {0, 2}), ("two_body_press", 2, {0, 1})):
        cfg = rsc.load_scene(os.path.join(ref_scenes, name + ".scn"))
        from dataclasses import replace

        cfg = replace(cfg, newton=replace(cfg.newton, scheme="fast", max_iterations=4,
                                          penetration_tol=-1.0, rotation_tol=-1.0),
                      pgs=replace(cfg.pgs, max_iterations=300, tolerance=1e-10),
                      output=rsc.OutputConfig(snapshots=False, metrics=False))
        out = _run_scene(cfg, steps, cap, tag=name)
        for obj in rsc.Simulation(cfg).dynamic_objects:
            out[f"mesh{obj.oid}_nodes"] = obj.spec.mesh.nodes
            out[f"mesh{obj.oid}_tets"] = obj.spec.mesh.tets
            out[f"mat{obj.oid}"] = np.array([obj.spec.young, obj.spec.poisson, obj.spec.density,
                                             obj.spec.rayleigh_mass, obj.spec.rayleigh_stiffness])
            out[f"vel{obj.oid}"] = np.array(obj.spec.velocity)
        save(f"{name}.npz", **out)


def beam_cfg0_full():
    """BASELINE cfg0 exactly as specified: 100 steps from 2 cm above the plane,
    jitter from default_rng(0).  Per-step pair counts, Newton iterations, PGS
    sweeps and pen_after; q and v every 10 steps and at the end."""
    cfg, mesh = beam_cfg0(drop=0.02)
    sim = rsc.Simulation(cfg)
    rng = np.random.default_rng(0)
    obj = sim.dynamic_objects[0]
    obj.state.q = obj.state.q + rng.uniform(-1e-4, 1e-4, obj.state.q.shape)
    npairs, newton, sweeps, pen = [], [], [], []
    out = {}
    for s in range(100):
        rep = sim.step()
        npairs.append(rep.c_groups)
        newton.append(rep.newton_iterations)
        sweeps.append(rep.pgs_iterations_total)
        pen.append(rep.pen_after)
        if s % 10 == 9:
            out[f"q{s}"], out[f"v{s}"] = obj.state.q.copy(), obj.state.v.copy()
            print("beam100 step", s, "pairs", rep.c_groups, "pgs", rep.pgs_iterations_total, flush=True)
    out.update(npairs=np.array(npairs), newton=np.array(newton), sweeps=np.array(sweeps), pen_after=np.array(pen),
               nodes=mesh.nodes, tets=mesh.tets, normal=np.array(cfg.objects[1].normal))
    save("beam_cfg0_100.npz", **out)


def cfg1_parity():
    """BASELINE cfg1 (isolated compliance-update bench) run by the reference
    itself: n = 12 000 (40x10x10-node 5-tet grid), 500 barycentric contacts,
    W_g = S A^-1 S^T (assemble_Wg constraints.py:155-179), then 10 frame
    re-draws: W_k = D_k W_g D_k^T (rebuild_W_fast 182-191, naive gemm) and
    dx_k = h A^-1 S^T D_k^T lam_k (_mechanical_correction solver.py:250-257).
    The inputs come from workloads.cfg1_inputs (the benched workload).  Stored:
    sampled rows of W_g and every W_k, the products W_g r and W_k r for a fixed
    random r (every entry enters), and dx_k (3 in full, every k sampled)."""
    import workloads as wk

    inp = wk.cfg1_inputs()
    nodes = inp["nodes"]
    body = cn.SoftBody(cn.TetMesh(nodes, inp["tets"]), young=5e3, poisson=0.45, density=1000.0,
                       rayleigh_mass=0.0, rayleigh_stiffness=0.0)
    st = body.initial_state()
    A, _ = body.assemble(st, wk.H, (0.0, -9.81, 0.0))
    F = cn.factorize(A)
    pairs = []
    for i in range(wk.CFG1_CONTACTS):
        tri = inp["tris"][inp["tri_idx"][i]]
        w = inp["weights"][i]
        p = w @ nodes[tri]
        pairs.append(rcol.ProximityPair(
            0, 1, rcol.Attachment(rcol.AttachKind.BARYCENTRIC, 0, triangle=tri.copy(), weights=w.copy()),
            rcol.Attachment(rcol.AttachKind.WORLD, 1, world_point=p.copy()), p.copy(), p.copy(),
            np.array([0.0, 1.0, 0.0]), 0.0, i, int(inp["tri_idx"][i])))
    S = rcon.build_signed_mapping(pairs, 0, body.n_dofs, body.fixed_mask)
    wg = rcon.assemble_Wg({0: S}, {0: F})
    m = 3 * wk.CFG1_CONTACTS
    rng = np.random.default_rng(11)
    rows = np.sort(rng.choice(m, 32, replace=False))
    r = rng.standard_normal(m)
    dsel = np.sort(rng.choice(body.n_dofs, 600, replace=False))
    out = dict(rows=rows, r=r, dsel=dsel, wg_rows=wg.wg[rows], wg_r=wg.wg @ r,
               S_indptr=S.indptr, S_indices=S.indices, S_data=S.data)
    for k in range(wk.CFG1_REDRAWS):
        frames = [rcol.ContactFrame(n=f[0], t1=f[1], t2=f[2]) for f in inp["Ds"][k]]
        D = rcon.assemble_direction(frames)
        W = rcon.rebuild_W_fast(D, wg).W
        out[f"W{k}_rows"], out[f"W{k}_r"] = W[rows[:8]], W @ r
        t = D.apply_transposed(inp["lams"][k])
        dx = wk.H * F.solve(S.T @ t)
        out[f"dx{k}_sel"] = dx[dsel]
        if k in (0, 4, 9):
            out[f"dx{k}"] = dx
        print("cfg1 redraw", k, flush=True)
    save("cfg1_parity.npz", **out)


def scenes_standard():
    """Reference runs of the standard (Alg. 2) and single schemes on block_on_plane."""
    from dataclasses import replace

    ref_scenes = "/root/reference/pkg/scenes"
    base = rsc.load_scene(os.path.join(ref_scenes, "block_on_plane.scn"))
    for scheme, iters in (("standard", 3), ("single", 1)):
        cfg = replace(base, newton=replace(base.newton, scheme=scheme, max_iterations=iters, penetration_tol=-1.0,
                                           rotation_tol=-1.0),
                      pgs=replace(base.pgs, max_iterations=300, tolerance=1e-10),
                      output=rsc.OutputConfig(snapshots=False, metrics=False))
        sim = rsc.Simulation(cfg)
        out = {}
        for s in range(2):
            rep = sim.step()
            out[f"s{s}_npairs"] = rep.c_groups
            out[f"s{s}_newton"] = rep.newton_iterations
            out[f"s{s}_lam"] = sim.last_lam.copy()
            for obj in sim.dynamic_objects:
                out[f"s{s}_q{obj.oid}"] = obj.state.q.copy()
            print(scheme, "step", s, "pairs", rep.c_groups, "newton", rep.newton_iterations)
        save(f"block_on_plane_{scheme}.npz", **out)


def kat_linalg():
    rng = np.random.default_rng(400)
    mesh = cn.box_mesh((0.1, 0.1, 0.1), (2, 2, 2), (0.0, 0.05, 0.0))
    body = cn.SoftBody(mesh, young=5e4, poisson=0.3, fixed_nodes=np.array([0, 1, 2]))
    st = body.initial_state((0.1, -0.2, 0.0))
    A, b = body.assemble(st, 0.01, (0.0, -9.81, 0.0))
    F = cn.factorize(A)
    x = F.solve(b)
    B = rng.standard_normal((A.dim, 5))
    X = F.solve_multi(B)
    csr = A.csr
    K = body.stiffness()
    save("kat_linalg.npz", nodes=mesh.nodes, tets=mesh.tets, indptr=csr.indptr, indices=csr.indices,
         data=csr.data, b=b, x=x, B=B, X=X, q=st.q, v=st.v, K_indptr=K.indptr, K_indices=K.indices,
         K_data=K.data, masses=body.masses())


def ellipsoid_mesh(semi=(0.05, 0.03, 0.025), spacing=0.008, seed=0):
    """Small cfg2-style body: jittered lattice inside an ellipsoid, Delaunay tets,
    centroid-inside / sliver filter, positive orientation."""
    from scipy.spatial import Delaunay

    rng = np.random.default_rng(seed)
    a = np.asarray(semi)
    axes = [np.arange(-ai, ai + 1e-12, spacing) for ai in a]
    P = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    P = P + rng.uniform(-0.25 * spacing, 0.25 * spacing, P.shape)
    P = P[((P / a) ** 2).sum(axis=1) <= 1.0]
    tri = Delaunay(P)
    T = tri.simplices.astype(np.int64)
    cen = P[T].mean(axis=1)
    T = T[((cen / a) ** 2).sum(axis=1) <= 1.0]
    v = np.einsum("ij,ij->i", np.cross(P[T[:, 1]] - P[T[:, 0]], P[T[:, 2]] - P[T[:, 0]]), P[T[:, 3]] - P[T[:, 0]]) / 6
    T[v < 0] = T[v < 0][:, [0, 2, 1, 3]]
    T = T[np.abs(v) >= 1e-3 * spacing ** 3]
    used = np.unique(T)
    remap = -np.ones(len(P), dtype=np.int64)
    remap[used] = np.arange(len(used))
    return P[used], remap[T]


def cylinder_surface(radius=0.015, length=0.06, n_theta=24, n_z=6):
    """Open cylinder (side surface) along z through the origin, outward wound."""
    th = np.linspace(0.0, 2 * np.pi, n_theta, endpoint=False)
    zs = np.linspace(-0.5 * length, 0.5 * length, n_z + 1)
    pts = np.array([[radius * np.cos(t), radius * np.sin(t), z] for z in zs for t in th])
    tris = []
    for k in range(n_z):
        for j in range(n_theta):
            a, b = k * n_theta + j, k * n_theta + (j + 1) % n_theta
            c, d = a + n_theta, b + n_theta
            tris += [[a, b, d], [a, d, c]]
    tris = np.array(tris, dtype=np.int64)
    n0 = np.cross(pts[tris[:, 1]] - pts[tris[:, 0]], pts[tris[:, 2]] - pts[tris[:, 0]])
    out = pts[tris].mean(axis=1) * np.array([1.0, 1.0, 0.0])
    flip = np.einsum("ij,ij->i", n0, out) < 0
    tris[flip] = tris[flip][:, ::-1]
    return pts, tris


def cylinder_press():
    """cfg2-style reference run: soft ellipsoid with its bottom 5 % fixed, pressed by a
    rigid cylinder rotating at 1 rad/s about its own axis (kinematic mesh), mu = 0.3,
    forced fast-scheme iterations with re-linearisation."""
    nodes, tets = ellipsoid_mesh()
    fixed = np.argsort(nodes[:, 1], kind="stable")[: max(1, len(nodes) // 20)]
    top = float(nodes[:, 1].max())
    pts, tris = cylinder_surface()
    center = (0.0, top + 0.015 - 0.003, 0.0)  # 3 mm indentation
    soft = rsc.SoftSpec(name="ellipsoid", mesh=cn.TetMesh(nodes, tets), young=3e3, poisson=0.45, density=1000.0,
                        fixed_nodes=np.sort(fixed))
    cyl = rsc.KinematicMeshSpec(name="cylinder", points=pts + np.asarray(center), triangles=tris,
                                motion=rsc.MotionSpec(axis=(0.0, 0.0, 1.0), center=center, angular_velocity=1.0))
    cfg = rsc.SceneConfig(objects=[soft, cyl], h=0.01, threshold=0.004,
                          pgs=rsol.PgsConfig(max_iterations=400, tolerance=1e-10, friction=0.3),
                          newton=rsol.NewtonConfig(scheme="fast", max_iterations=4, penetration_tol=-1,
                                                   rotation_tol=-1),
                          output=rsc.OutputConfig(snapshots=False, metrics=False))
    out = _run_scene(cfg, 3, {0, 2}, tag="cylinder_press")
    out.update(nodes=nodes, tets=tets, fixed=np.sort(fixed), cyl_points=pts + np.asarray(center), cyl_tris=tris,
               center=np.asarray(center))
    save("cylinder_press.npz", **out)


SCENE_IO_TEXT = """\
# scene-format fixture: soft box on the ground, pushed by a moving plate
gravity: [0.0, -9.81, 0.0]
dt: 0.01
threshold: 0.008
mu: 0.4
pgs: {iterations: 150, tolerance: 1.0e-8}
newton: {scheme: fast, iterations: 3, penetration_tol: -1.0}
output: {snapshots: true, metrics: true, every: 1}
objects:
  - name: cube
    type: soft
    mesh: {box: {size: [0.04, 0.04, 0.04], divisions: [3, 3, 3], center: [0.0, 0.0205, 0.0]}}
    material: {young: 3.0e4, poisson: 0.35, density: 900.0, rayleigh_mass: 0.1, rayleigh_stiffness: 0.05}
    velocity: [0.1, 0.0, 0.0]
  - name: ground
    type: plane
    normal: [0.0, 1.0, 0.0]
    offset: 0.0
  - name: pusher
    type: kinematic_mesh
    plate: {center: [0.03, 0.02, 0.0], normal: [-1.0, 0.0, 0.0], size: [0.06, 0.06]}
    motion: {velocity: [-0.05, 0.0, 0.0]}
"""


def scene_io():
    """Reference parse of a scene file, its metrics.csv and snapshot files after a
    3-step run (scene.py:292-354, 541-547, 771-866)."""
    import json
    import shutil
    import tempfile

    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "io.scn")
    with open(path, "w") as fh:
        fh.write(SCENE_IO_TEXT)
    cfg = rsc.load_scene(path)
    summary = {"h": cfg.h, "threshold": cfg.threshold, "gravity": list(cfg.gravity),
               "pgs": [cfg.pgs.max_iterations, cfg.pgs.tolerance, cfg.pgs.friction],
               "newton": [cfg.newton.scheme, cfg.newton.max_iterations, cfg.newton.penetration_tol,
                          cfg.newton.relinearize],
               "output": [cfg.output.snapshots, cfg.output.metrics, cfg.output.every], "objects": []}
    arrays = {}
    for k, o in enumerate(cfg.objects):
        d = {"name": o.name, "type": type(o).__name__}
        if hasattr(o, "mesh"):
            d.update(young=o.young, poisson=o.poisson, density=o.density, rayleigh_mass=o.rayleigh_mass,
                     rayleigh_stiffness=o.rayleigh_stiffness, velocity=list(o.velocity))
            arrays[f"nodes{k}"], arrays[f"tets{k}"] = o.mesh.nodes, o.mesh.tets
        elif hasattr(o, "points"):
            d.update(axis=list(o.motion.axis), center=list(o.motion.center),
                     angular_velocity=o.motion.angular_velocity, velocity=list(o.motion.velocity))
            arrays[f"points{k}"], arrays[f"triangles{k}"] = o.points, o.triangles
        else:
            d.update(normal=list(o.normal), offset=o.offset)
        summary["objects"].append(d)
    out_dir = os.path.join(tmp, "out")
    sim = rsc.Simulation(cfg)
    reps = rsc.run(sim, 3, out_dir)
    for r in reps:
        print("scene_io step", r.step, "pairs", r.c_groups, "newton", r.newton_iterations, "pgs", r.pgs_iterations_total)
    with open(os.path.join(HERE, "scene_io.scn"), "w") as fh:
        fh.write(SCENE_IO_TEXT)
    with open(os.path.join(HERE, "scene_io.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    shutil.copy(os.path.join(out_dir, "metrics.csv"), os.path.join(HERE, "scene_io_metrics.csv"))
    for st in (0, 2):
        shutil.copy(os.path.join(out_dir, "snapshots", f"step_{st:06d}.bin"),
                    os.path.join(HERE, f"scene_io_step_{st:06d}.bin"))
    save("scene_io.npz", **arrays)
    shutil.rmtree(tmp)


def fixed_mapping():
    """Two stacked five-tet blocks; the lower one rests on the ground with its
    bottom layer and part of its top face fixed, so vertex-plane and
    barycentric rows both land on fixed DoFs.  Records the reference's pair
    keys, the signed mappings S_o (build_signed_mapping constraints.py:101-120:
    fixed columns zeroed and dropped) and the system-matrix patterns
    (SoftBody.assemble dynamics.py:183-211: fixed rows/cols -> identity), then
    a 3-step forced fast-scheme trajectory."""
    lower = five_tet_grid((5, 3, 5), 0.01, (0.0, 0.0015, 0.0))
    upper = five_tet_grid((4, 2, 4), 0.01, (0.005, 0.0235, 0.005))
    ln = lower.nodes
    bottom = np.flatnonzero(ln[:, 1] <= ln[:, 1].min() + 1e-12)
    top = np.flatnonzero(ln[:, 1] >= ln[:, 1].max() - 1e-12)
    fixed_top = top[(ln[top, 0] <= 0.02 + 1e-12) & (ln[top, 2] <= 0.02 + 1e-12)]
    fixed = np.sort(np.concatenate([bottom, fixed_top]))
    soft0 = rsc.SoftSpec(name="lower", mesh=cn.TetMesh(lower.nodes, lower.tets), young=1e4, poisson=0.4,
                         density=1000.0, fixed_nodes=fixed)
    soft1 = rsc.SoftSpec(name="upper", mesh=cn.TetMesh(upper.nodes, upper.tets), young=2e3, poisson=0.4,
                         density=1000.0, velocity=(0.0, -0.1, 0.0))
    plane = rsc.PlaneSpec(name="ground", normal=(0.0, 1.0, 0.0), offset=0.0)
    cfg = rsc.SceneConfig(objects=[soft0, soft1, plane], h=0.01, threshold=0.004,
                          pgs=rsol.PgsConfig(max_iterations=400, tolerance=1e-10, friction=0.4),
                          newton=rsol.NewtonConfig(scheme="fast", max_iterations=3, penetration_tol=-1,
                                                   rotation_tol=-1),
                          output=rsc.OutputConfig(snapshots=False, metrics=False))
    sim = rsc.Simulation(cfg)
    out = {}
    ctx, free, states, pen_before, timings, t_next = sim.prepare_step(build_wg=True)
    for oid, S in ctx.S_by_object.items():
        S = S.tocsr()
        out[f"S{oid}_indptr"], out[f"S{oid}_indices"], out[f"S{oid}_data"] = S.indptr, S.indices, S.data
    for obj in sim.dynamic_objects:
        A, b = obj.body.assemble(obj.state, cfg.h, cfg.gravity)
        out[f"A{obj.oid}_indptr"], out[f"A{obj.oid}_indices"] = A.csr.indptr, A.csr.indices
        out[f"A{obj.oid}_data"], out[f"b{obj.oid}"] = A.csr.data, b
    out.update(_run_scene(cfg, 3, {0}, tag="fixed_mapping"))
    out.update(lower_nodes=lower.nodes, lower_tets=lower.tets, upper_nodes=upper.nodes, upper_tets=upper.tets,
               fixed=fixed)
    save("fixed_mapping.npz", **out)


def rigid_spheres():
    """Rigid spheres (dynamics.py:214-249, RIGID_LOCAL rows collision.py:448-457,
    sphere-plane pairs collision.py:290-316) on a tilted plane with friction,
    one spinning, beside a soft box that lands on the plane: 14 forced fast-scheme steps.  Per step the
    pair keys, Newton iterations, q / v of every dynamic object and the
    spheres' rotations."""
    ang = np.deg2rad(15.0)
    normal = (float(np.sin(ang)), float(np.cos(ang)), 0.0)
    box = cn.box_mesh((0.04, 0.04, 0.04), (2, 2, 2), (0.1, 0.045, 0.0))
    objs = [rsc.SoftSpec(name="box", mesh=box, young=2e4, poisson=0.3, density=800.0),
            rsc.RigidSphereSpec(name="ball", mass=0.3, radius=0.02, position=(0.0, 0.0215, 0.0),
                                velocity=(0.2, -0.3, 0.0, 0.0, 0.0, 4.0),
                                inertia=np.diag([1e-4, 1.2e-4, 0.8e-4])),
            rsc.RigidSphereSpec(name="marble", mass=0.05, radius=0.01, position=(-0.06, 0.012, 0.03),
                                velocity=(0.0, 0.0, 0.0, 0.0, 0.0, 0.0),
                                inertia=(0.4 * 0.05 * 0.01 ** 2) * np.eye(3)),
            rsc.PlaneSpec(name="ground", normal=normal, offset=0.0)]
    cfg = rsc.SceneConfig(objects=objs, h=0.01, threshold=0.006,
                          pgs=rsol.PgsConfig(max_iterations=500, tolerance=1e-11, friction=0.4),
                          newton=rsol.NewtonConfig(scheme="fast", max_iterations=3, penetration_tol=-1,
                                                   rotation_tol=-1),
                          output=rsc.OutputConfig(snapshots=False, metrics=False))
    sim = rsc.Simulation(cfg)
    out = {}
    for st in range(14):
        ctx, free, states, pen_before, timings, t_next = sim.prepare_step(build_wg=True)
        res = rsol.newton_fast(ctx, cfg.newton, cfg.pgs)
        out[f"s{st}_keys"] = np.array([(p.object_a, p.object_b, p.vertex_id, p.element_id) for p in ctx.pairs],
                                      dtype=np.int64).reshape(-1, 4)
        if ctx.pairs:
            out[f"s{st}_lamhist"] = np.stack(res.lam_history)
        rep = sim.step()
        out[f"s{st}_npairs"] = rep.c_groups
        out[f"s{st}_newton"] = rep.newton_iterations
        for obj in sim.dynamic_objects:
            out[f"s{st}_q{obj.oid}"] = obj.state.q.copy()
            out[f"s{st}_v{obj.oid}"] = obj.state.v.copy()
            if obj.kind == "rigid":
                out[f"s{st}_R{obj.oid}"] = obj.rotation.copy()
        print("rigid_spheres step", st, "pairs", rep.c_groups, "newton", rep.newton_iterations,
              "pgs", rep.pgs_iterations_total, flush=True)
    out.update(box_nodes=box.nodes, box_tets=box.tets, normal=np.array(normal))
    save("rigid_spheres.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kat_rebuild", "kat_pgs", "kat_frames", "kat_linalg", "scenes", "scenes_standard",
                             "scene_io", "cylinder_press"]
    for name in which:
        globals()[name]()
