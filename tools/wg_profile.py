"""Host/GPU split of the per-step compliance build on the cfg3 scene (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_06946_b200 import wg as wgm  # noqa: E402

wl = bench.Cfg3Workload()
wl.step()
torch.cuda.synchronize()
ctx = wl.sim.prepare_step(build_wg=False)[0]
torch.cuda.synchronize()
for rep in range(2):
    for oid in sorted(ctx.S_by_object):
        S, F = ctx.S_by_object[oid], ctx.F_by_object[oid]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U = wgm.object_compliance(S, F, 3 * len(ctx.pairs))
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"obj {oid}: mo={len(S.idx)} host-enqueue {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms", flush=True)
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for oid in sorted(ctx.S_by_object):
    wgm.object_compliance(ctx.S_by_object[oid], ctx.F_by_object[oid], 3 * len(ctx.pairs))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
