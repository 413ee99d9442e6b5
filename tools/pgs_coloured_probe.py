"""Exact-order vs graph-coloured PGS on the two-block scene's first W (step 1):
sweeps, time, convergence history and the difference of the converged lambda.
    python tools/pgs_coloured_probe.py [nxz ny]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06946_b200 as cn  # noqa: E402
from paper_2306_06946_b200.solver import colour_groups  # noqa: E402

nxz = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 5
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = bench.make_cfg3_config(cn, nxz=nxz, ny=ny, shift=bench.CFG3_SHIFT, gap=bench.CFG3_GAP)
sim = cn.Simulation(cfg)
for _ in range(steps):
    sim.step()
ctx = sim.prepare_step(build_wg=True)[0]
G = len(ctx.pairs)
D = cn.assemble_direction(ctx.detection_frames)
W = cn.rebuild_W_fast(D, ctx.wg).W
delta = cn.compute_violation(D, ctx.p_a0, ctx.p_b0).delta
colours = colour_groups(ctx.S_by_object, G)
print(json.dumps({"groups": G, "colours": len(colours[0]) - 1,
                  "colour_sizes": np.diff(colours[0]).tolist()[:40]}), flush=True)
res = {}
omegas = [float(x) for x in os.environ.get("OMEGAS", "0.5,0.2,0.05").split(",")]
runs = [("exact", {})] + [(f"coloured_w{w}", {"ordering": "coloured", "relaxation": w}) for w in omegas]
for name, kw in runs:
    for tol, mx in ((1e-6, 30), (1e-6, 3000), (1e-10, 20000)):
        pc = cn.PgsConfig(max_iterations=mx, tolerance=tol, friction=0.4, **kw)
        cn.pgs(W, delta, cfg.h, pc, colours=colours)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = cn.pgs(W, delta, cfg.h, pc, colours=colours)
        e1.record()
        torch.cuda.synchronize()
        eps = r.eps_history
        res[(name, tol, mx)] = r.lam.clone()
        print(json.dumps({"ordering": name, "tol": tol, "max": mx, "sweeps": r.iterations, "converged": r.converged,
                          "ms": round(e0.elapsed_time(e1), 3), "ms_per_sweep": round(e0.elapsed_time(e1) / r.iterations, 4),
                          "eps": [float(f"{x:.3e}") for x in (eps[:5] + eps[-3:])]}), flush=True)
a = res[("exact", 1e-10, 20000)]
for name, _ in runs[1:]:
    b = res[(name, 1e-10, 20000)]
    print(json.dumps({name: {"converged_lambda_rel_diff": float((a - b).abs().max() / a.abs().max())}}), flush=True)
