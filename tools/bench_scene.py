"""Scene-level benchmark: BASELINE configs[0] (cfg0 beam) through Simulation.step.

20x4x4-node 5-tet beam (960 DoF, E=5e3, nu=0.45, rho=1000, Rayleigh 0.1/0.1)
over a plane tilted 10 degrees, threshold 0.005, mu=0.5, 5 forced Newton
iterations (tolerances -1), PGS to 1e-10 (<= 1000 sweeps), jitter U(-1e-4,1e-4)
from rng 0.  The beam starts 2 mm above the plane so contacts exist after a
few warm-up steps.  Prints one JSON line: ms per step, ms per Newton
iteration (rebuild W + PGS + proximity update), PGS sweeps, and the CPU
oracle port on a bounded sample (--cpu-steps).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def beam(drop=0.002):
    from paper_2306_06946_b200.mesh import five_tet_grid

    ang = np.deg2rad(10.0)
    normal = np.array([np.sin(ang), np.cos(ang), 0.0])
    mesh = five_tet_grid((20, 4, 4), 0.01, (0.0, drop / normal[1], 0.0))
    return mesh, normal


def gpu_run(args):
    import torch

    import paper_2306_06946_b200 as cn

    mesh, normal = beam()
    cfg = cn.SceneConfig(
        objects=[cn.SoftSpec(name="beam", mesh=mesh, young=5e3, poisson=0.45, density=1000.0,
                             material=args.material),
                 cn.PlaneSpec(name="ground", normal=tuple(normal), offset=0.0)],
        threshold=0.005, pgs=cn.PgsConfig(1000, 1e-10, 0.5),
        newton=cn.NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0, rotation_tol=-1.0),
        output=cn.OutputConfig(snapshots=False, metrics=False))
    sim = cn.Simulation(cfg)
    rng = np.random.default_rng(0)
    st = sim.objects[0].state
    sim.objects[0].state = cn.MechanicalState(st.q.cpu().numpy() + rng.uniform(-1e-4, 1e-4, st.q.shape[0]), st.v)
    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    reps = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        reps.append(sim.step())
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / args.steps
    it_ms = [1e3 * (r + p + c) for rep in reps for r, p, c in
             zip(rep.rebuild_times, rep.pgs_times, rep.correction_times)]
    pgs_ms = [1e3 * p for rep in reps for p in rep.pgs_times]
    phases = {f"{k}_ms": 1e3 * statistics.median(getattr(r, k) for r in reps) for k in
              ("t_detect", "t_assemble", "t_free", "t_constraints", "t_build_wg", "t_rebuild_w", "t_pgs",
               "t_correction", "t_final_correction", "t_step")}
    print(json.dumps({"phases_median": {k: round(v, 3) for k, v in phases.items()}}), flush=True)
    return dict(ms_per_step=wall, ms_per_newton_iter=statistics.median(it_ms), pgs_ms_median=statistics.median(pgs_ms),
                pgs_sweeps_per_step=statistics.mean(r.pgs_iterations_total for r in reps),
                groups=statistics.mean(r.c_groups for r in reps), t_detect_ms=1e3 * statistics.median(
                    r.t_detect for r in reps), t_build_wg_ms=1e3 * statistics.median(r.t_build_wg for r in reps))


def cpu_run(steps, warmup):
    import cn_oracle as orc

    mesh, normal = beam()
    body = orc.Body(mesh.nodes, mesh.tets, young=5e3, poisson=0.45, density=1000.0)
    sc = orc.Scene([body], [dict(normal=normal, offset=0.0)], threshold=0.005, mu=0.5, pgs_iter=1000,
                   pgs_tol=1e-10, newton_iter=5, penetration_tol=-1.0, rotation_tol=-1.0)
    rng = np.random.default_rng(0)
    sc.q[0] = sc.q[0] + rng.uniform(-1e-4, 1e-4, sc.q[0].shape)
    for _ in range(warmup):
        sc.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        sc.step()
    return (time.perf_counter() - t0) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--material", default="linear")
    args = ap.parse_args()
    g = gpu_run(args)
    line = {"metric": "cfg0 beam: ms per full step / per Newton iteration (fast scheme, PGS to 1e-10)",
            "unit": "ms", "material": args.material, "gpu": {k: round(v, 4) for k, v in g.items()}}
    if args.cpu_steps > 0:
        cpu_ms = cpu_run(args.cpu_steps, args.warmup)
        line["cpu_oracle_port_ms_per_step"] = round(cpu_ms, 1)
        line["cpu_sample"] = f"{args.cpu_steps} steps after {args.warmup} warm-up steps, same scene and seeds"
        line["speedup_step"] = round(cpu_ms / g["ms_per_step"], 1)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
