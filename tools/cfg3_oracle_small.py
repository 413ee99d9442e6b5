"""The cfg3 scene at reduced size through the CPU oracle (reference algorithm,
linear or corotational material), to show its dynamics: penetration and contact
count per step.  With the BASELINE materials (upper block E = 2 kPa) the
reference algorithm itself degenerates after a few steps, as the GPU run does
at full size (tools/cfg3_steps.py).  Test infrastructure: runs on the CPU.

    python tools/cfg3_oracle_small.py NXZ NY SHIFT GAP PGS_SWEEPS STEPS [corot]
    e.g. python tools/cfg3_oracle_small.py 8 6 0.005 0.001 30 10 corot
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import cn_oracle as orc  # noqa: E402
import workloads as wk  # noqa: E402

nxz, ny = int(sys.argv[1]), int(sys.argv[2])
shift, gap = float(sys.argv[3]), float(sys.argv[4])
sweeps, steps = int(sys.argv[5]), int(sys.argv[6])
B = orc.CorotBody if "corot" in sys.argv[7:] else orc.Body
(ln, lt), (un, ut) = wk.cfg3_meshes(nxz, ny, shift, gap)
bodies = [B(ln, lt, young=1e4, poisson=0.4), B(un, ut, young=2e3, poisson=0.4)]
sc = orc.Scene(bodies, [dict(normal=(0.0, 1.0, 0.0), offset=0.0)], threshold=0.005, mu=0.4, pgs_iter=sweeps,
               pgs_tol=1e-6, newton_iter=10, penetration_tol=-1, rotation_tol=-1,
               velocities=[(0, 0, 0), (0.5, 0, 0)])
for s in range(steps):
    t = time.time()
    out = sc.step()
    print(s, out["n_pairs"], "pen_before %.3e pen_after %.3e" % (out["pen_before"], out["pen_after"]),
          "sweeps", sum(out["result"]["pgs_iterations"]) if "result" in out else 0, "%.1fs" % (time.time() - t),
          flush=True)
