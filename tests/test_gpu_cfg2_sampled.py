"""BASELINE cfg2 at full size (soft ellipsoid of ~29 000 nodes / 88 000 DoF, bottom
5 % fixed, pressed by a rigid cylinder rotating at 1 rad/s, mu = 0.3, 10
re-linearised fast iterations, PGS 30 sweeps / tol 1e-6), where a reference run
of a whole step is out of reach (dense S^T / X, naive-gemm rebuilds): sampled,
size-independent checks after one step, as for cfg3 (test_gpu_cfg3_sampled.py):

* W_g columns: solves on the GPU factor for sampled rows of S, residual against
  the CPU oracle's own A (reference formulas, linear material) <= 1e-12, and the
  GPU's W_g columns = S x within 1e-9;
* the first Newton iteration's PGS (fixed budget) against the oracle's
  restatement of the reference pgs on the downloaded W (lambda within 1e-6,
  same sweep count) and the same lambda inside newton_fast.
"""

import numpy as np
import pytest
import torch

import cn_oracle as orc
import workloads

pytestmark = pytest.mark.gpu


def _h(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.fixture(scope="module")
def scene():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_06946_b200 as cn

    nodes, tets, fixed, pts, tris, center = workloads.cfg2_arrays()
    soft = cn.SoftSpec(name="ellipsoid", mesh=cn.TetMesh(nodes, tets), young=3e3, poisson=0.45, density=1000.0,
                       fixed_nodes=fixed)
    cyl = cn.KinematicMeshSpec(name="cylinder", points=pts, triangles=tris,
                               motion=cn.MotionSpec(axis=(0.0, 0.0, 1.0), center=tuple(center), angular_velocity=1.0))
    cfg = cn.SceneConfig(objects=[soft, cyl], h=0.01, threshold=0.004,
                         pgs=cn.PgsConfig(max_iterations=30, tolerance=1e-6, friction=0.3),
                         newton=cn.NewtonConfig(scheme="fast", max_iterations=10, penetration_tol=-1.0,
                                                rotation_tol=-1.0),
                         output=cn.OutputConfig(snapshots=False, metrics=False))
    sim = cn.Simulation(cfg)
    rep = sim.step()
    ctx = sim.prepare_step(build_wg=True)[0]
    return cn, cfg, sim, rep, ctx, (nodes, tets, fixed)


def test_scene_runs_at_baseline_size(scene):
    cn, cfg, sim, rep, ctx, (nodes, tets, fixed) = scene
    assert sim.total_dofs() == 3 * len(nodes) > 80000
    assert rep.newton_iterations == 10 and rep.c_groups > 100
    q = _h(sim.objects[0].state.q).reshape(-1, 3)
    assert np.array_equal(q[fixed], nodes[fixed])  # fixed nodes stay (zero initial velocity)


def test_compliance_columns_against_oracle_system(scene):
    cn, cfg, sim, rep, ctx, (nodes, tets, fixed) = scene
    wg = _h(ctx.wg.wg)
    obj = sim.dynamic_objects[0]
    S = ctx.S_by_object[obj.oid].sorted_csr
    rng = np.random.default_rng(7)
    pick = np.sort(rng.choice(wg.shape[0], 8, replace=False))
    B = S[pick].toarray().T
    X = _h(ctx.F_by_object[obj.oid].solve_multi(B))
    ob = orc.Body(nodes, tets, young=3e3, poisson=0.45, density=1000.0, fixed_nodes=fixed)
    A, _ = ob.system(_h(obj.state.q), _h(obj.state.v), cfg.h, cfg.gravity)
    assert np.abs(A @ X - B).max() <= 1e-12 * np.abs(B).max()
    ref = S @ X
    assert np.abs(wg[:, pick] - ref).max() <= 1e-9 * np.abs(ref).max()


def test_pgs_first_iteration_against_oracle(scene):
    cn, cfg, sim, rep, ctx, _ = scene
    D = cn.assemble_direction(ctx.detection_frames)
    W = cn.rebuild_W_fast(D, ctx.wg).W
    delta = cn.compute_violation(D, ctx.p_a0, ctx.p_b0).delta
    res = cn.pgs(W, delta, cfg.h, cfg.pgs)
    lam_gpu = _h(res.lam)
    lam, dend, it, hist, conv = orc.pgs(_h(W), _h(delta), cfg.h, max_iter=cfg.pgs.max_iterations,
                                        tol=cfg.pgs.tolerance, mu=cfg.pgs.friction)
    scale = np.abs(lam).max()
    assert np.abs(lam_gpu - lam).max() <= 1e-6 * scale
    assert res.iterations == it
    r = cn.newton_fast(ctx, cfg.newton, cfg.pgs)
    assert np.abs(_h(r.lam_history[0]) - lam_gpu).max() <= 1e-12 * scale
