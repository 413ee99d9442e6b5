"""Parity of the benched BASELINE cfg3 scene (450 000 DoF, two corotational
blocks, ~7 500 contact groups) at full size, where no CPU run of the whole step
is feasible: size-independent checks on sampled pieces.

* X columns: A_o x = s_j solved on the GPU factor for sampled rows s_j of S_o;
  the residual against the CPU corotational oracle's own A_o (an independent
  assembly, oracle/cn_oracle.py CorotBody) is <= 1e-12 relative, and the
  GPU's W_g columns equal S x_j within 1e-9 (the Gram/sandwich path against
  plain solves).
* PGS: the 7 500-group pipelined kernel (pgs_pipe_kernel) on the step's first
  W = D W_g D^T against the oracle's restatement of the reference pgs
  (solver.py:168-202) on the downloaded W, same budget (30 sweeps, tol 1e-6):
  lambda within 1e-6, identical sweep count, and the same lambda as the
  first Newton iteration of newton_fast.
"""

import numpy as np
import pytest
import torch

import cn_oracle as orc

pytestmark = pytest.mark.gpu


def _h(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.fixture(scope="module")
def scene():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    import paper_2306_06946_b200 as cn

    cfg = bench.make_cfg3_config(cn)
    sim = cn.Simulation(cfg)
    sim.step()  # one step in: the upper block is sliding
    ctx = sim.prepare_step(build_wg=True)[0]
    return cn, cfg, sim, ctx


def test_compliance_columns_against_oracle_system(scene):
    cn, cfg, sim, ctx = scene
    wg = _h(ctx.wg.wg)
    rng = np.random.default_rng(5)
    objs = sim.dynamic_objects
    Ss = {o.oid: ctx.S_by_object[o.oid].sorted_csr for o in objs}
    # sampled rows j: W_g[:, j] = sum_o S_o A_o^-1 S_o[j, :]^T
    pick = np.sort(rng.choice(wg.shape[0], 8, replace=False))
    total = np.zeros((wg.shape[0], len(pick)))
    for obj in objs:
        oid = obj.oid
        S = Ss[oid]
        B = S[pick].toarray().T  # (n_o, 8)
        if not B.any():
            continue
        X = _h(ctx.F_by_object[oid].solve_multi(B))
        spec = cfg.objects[oid]
        ob = orc.CorotBody(spec.mesh.nodes, spec.mesh.tets, young=spec.young, poisson=spec.poisson,
                           density=spec.density)
        A, _ = ob.system(_h(obj.state.q), _h(obj.state.v), cfg.h, cfg.gravity)
        assert np.abs(A @ X - B).max() <= 1e-12 * np.abs(B).max(), oid
        total += S @ X
    assert np.abs(wg[:, pick] - total).max() <= 1e-9 * np.abs(total).max()


def test_pipelined_pgs_7500_groups_against_oracle(scene):
    cn, cfg, sim, ctx = scene
    G = len(ctx.pairs)
    assert G >= 7000
    D = cn.assemble_direction(ctx.detection_frames)
    W = cn.rebuild_W_fast(D, ctx.wg).W
    delta = cn.compute_violation(D, ctx.p_a0, ctx.p_b0).delta
    res = cn.pgs(W, delta, cfg.h, cfg.pgs)
    lam_gpu = _h(res.lam)
    Wh, dh = _h(W), _h(delta)
    del W
    torch.cuda.empty_cache()
    lam, dend, it, hist, conv = orc.pgs(Wh, dh, cfg.h, max_iter=cfg.pgs.max_iterations, tol=cfg.pgs.tolerance,
                                        mu=cfg.pgs.friction)
    scale = np.abs(lam).max()
    assert np.abs(lam_gpu - lam).max() <= 1e-6 * scale
    assert res.iterations == it
    assert np.abs(_h(res.delta_end) - dend).max() <= 1e-6 * np.abs(dend).max()
    # the Newton loop's first iteration runs the same PGS on the same W
    r = cn.newton_fast(ctx, cfg.newton, cfg.pgs)
    assert np.abs(_h(r.lam_history[0]) - lam_gpu).max() <= 1e-12 * scale
