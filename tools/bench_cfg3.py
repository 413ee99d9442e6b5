"""cfg3 scene probe: builds the two-block scene (bench.make_cfg3_config) and runs
whole Simulation.step() calls, printing the per-phase breakdown per step.

    python tools/bench_cfg3.py --nxz 50 --ny 30 --steps 3
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nxz", type=int, default=50)
    ap.add_argument("--ny", type=int, default=30)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2306_06946_b200 as cn
    from paper_2306_06946_b200 import _lib

    t0 = time.perf_counter()
    cfg = bench.make_cfg3_config(cn, args.nxz, args.ny)
    sim = cn.Simulation(cfg)
    print(json.dumps({"setup_s": round(time.perf_counter() - t0, 2), "dofs": sim.total_dofs()}), flush=True)
    for s in range(args.steps):
        torch.cuda.synchronize()
        l0 = _lib.lib().cnb_launch_count()
        t1 = time.perf_counter()
        rep = sim.step()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t1
        out = {"step": s, "wall_ms": round(wall * 1e3, 1), "pairs": rep.c_groups,
               "newton": rep.newton_iterations, "pgs_total": rep.pgs_iterations_total,
               "launches": int(_lib.lib().cnb_launch_count() - l0)}
        for k in ("t_detect", "t_assemble", "t_free", "t_constraints", "t_build_wg", "t_rebuild_w", "t_pgs",
                  "t_correction", "t_final_correction", "t_step"):
            out[k] = round(getattr(rep, k) * 1e3, 2)
        out["pen_before"], out["pen_after"] = rep.pen_before, rep.pen_after
        print(json.dumps(out), flush=True)
    F = [o.factorization for o in sim.dynamic_objects]
    print(json.dumps({"nnz_L": [f.nnz_L for f in F], "gflop": [round(f.flops / 1e9, 1) for f in F],
                      "front_gb": [round(f.front_doubles * 8 / 1e9, 2) for f in F],
                      "mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
