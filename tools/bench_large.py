"""Large-scene kernel benchmark (BASELINE configs[3] scale): one corotational
5-tet block, N seeded barycentric surface contacts, one compliance build and
Newton iterations (rebuild W + PGS 30 sweeps tol 1e-6 + proximity update).

    python tools/bench_large.py --shape 50 50 20 --contacts 8000
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=[50, 50, 20])
    ap.add_argument("--contacts", type=int, default=8000)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--sweeps", type=int, default=30)
    args = ap.parse_args()
    import torch

    import paper_2306_06946_b200 as cn
    from paper_2306_06946_b200 import _lib
    from paper_2306_06946_b200.constraints import prox_update_inplace
    from paper_2306_06946_b200.solver import pgs_device

    out = {"shape": args.shape, "contacts": args.contacts}
    t0 = time.perf_counter()
    mesh = cn.five_tet_grid(tuple(args.shape), 0.01)
    body = cn.SoftBody(mesh, young=1e4, poisson=0.4, density=1000.0, material="corotational")
    out["dofs"] = body.n_dofs
    tris = cn.surface_triangles(mesh)
    rng = np.random.default_rng(1)
    m = args.contacts
    tri_idx = rng.integers(0, len(tris), m)
    wts = rng.dirichlet((1.0, 1.0, 1.0), m)
    pairs = []
    for i in range(m):
        tri = tris[tri_idx[i]]
        p = wts[i] @ mesh.nodes[tri]
        pairs.append(cn.ProximityPair(0, 1, cn.Attachment(cn.AttachKind.BARYCENTRIC, 0, triangle=tri.copy(),
                                                          weights=wts[i].copy()),
                                      cn.Attachment(cn.AttachKind.WORLD, 1, world_point=p.copy()), p.copy(),
                                      p.copy(), np.array([0.0, 1.0, 0.0]), 0.0, i, int(tri_idx[i])))
    out["host_setup_s"] = round(time.perf_counter() - t0, 2)
    state = body.initial_state()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    A, b = body.assemble(state, 0.01, (0.0, -9.81, 0.0))
    F = cn.Factorization(A)
    torch.cuda.synchronize()
    out["first_factor_incl_analysis_s"] = round(time.perf_counter() - t1, 2)
    out["nnz_L"] = F.nnz_L
    out["factor_gflop"] = round(F.flops / 1e9, 1)
    out["front_gb"] = round(F.front_doubles * 8 / 1e9, 2)
    S = cn.build_signed_mapping(pairs, 0, body.n_dofs, body.fixed_mask)
    # timed: assemble + refactor, compliance
    e = [ev() for _ in range(4)]
    e[0].record()
    A, b = body.assemble(state, 0.01, (0.0, -9.81, 0.0))
    e[1].record()
    F.refactor_async(A.values)
    e[2].record()
    wg = cn.assemble_Wg({0: S}, {0: F})
    e[3].record()
    torch.cuda.synchronize()
    out["assemble_ms"] = round(e[0].elapsed_time(e[1]), 3)
    out["factor_ms"] = round(e[1].elapsed_time(e[2]), 3)
    out["build_wg_ms"] = round(e[2].elapsed_time(e[3]), 3)
    out["factor_tflops"] = round(F.flops / (e[1].elapsed_time(e[2]) * 1e-3) / 1e12, 3)
    # Newton iterations with random frames / violations
    c = 3 * m
    rngf = np.random.default_rng(2)
    n_ = rngf.standard_normal((m, 3))
    n_ /= np.linalg.norm(n_, axis=1, keepdims=True)
    t1v = np.cross(n_, rngf.standard_normal((m, 3)))
    t1v /= np.linalg.norm(t1v, axis=1, keepdims=True)
    D = torch.as_tensor(np.stack([n_, t1v, np.cross(n_, t1v)], axis=1), device="cuda")
    p_a = torch.as_tensor(np.stack([p.p_a for p in pairs]), device="cuda")
    p_b = p_a - torch.as_tensor(rngf.uniform(-1e-3, 1e-3, (m, 3)), device="cuda")
    W = torch.empty((c, c), dtype=torch.float64, device="cuda")
    delta = torch.empty(c, dtype=torch.float64, device="cuda")
    t = torch.empty(c, dtype=torch.float64, device="cuda")
    pcfg = cn.PgsConfig(args.sweeps, 1e-6, 0.4)
    times = []
    for k in range(args.iters):
        e = [ev() for _ in range(4)]
        e[0].record()
        cn.rebuild_W_fast(cn.DirectionMatrix(D), wg, out=W)
        e[1].record()
        cn.compute_violation(cn.DirectionMatrix(D), p_a, p_b, out=delta)
        res = pgs_device(W, delta, 0.01, pcfg)
        e[2].record()
        _lib.call("cnb_apply_dt", m, D.data_ptr(), res.lam.data_ptr(), t.data_ptr(), None, _lib.stream())
        prox_update_inplace(p_a, p_b, wg, t, 0.01)
        e[3].record()
        torch.cuda.synchronize()
        times.append([e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])])
        out["pgs_sweeps"] = res.iterations
    tm = np.median(np.array(times), axis=0)
    out["rebuild_w_ms"] = round(float(tm[0]), 3)
    out["pgs_ms"] = round(float(tm[1]), 3)
    out["prox_ms"] = round(float(tm[2]), 3)
    out["newton_iter_ms"] = round(float(tm.sum()), 3)
    out["rebuild_w_gbs"] = round(16.0 * c * c / (tm[0] * 1e-3) / 1e9, 1)
    out["pgs_gbs_per_sweep"] = round(8.0 * c * c * res.iterations / (tm[1] * 1e-3) / 1e9, 1)
    out["launches_total"] = int(_lib.lib().cnb_launch_count())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
