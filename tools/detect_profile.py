"""Host profile of one cfg3 step's detection phase (where the 'detect' time goes)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_06946_b200 import collision  # noqa: E402

wl = bench.Cfg3Workload()
wl.step()
torch.cuda.synchronize()
sim = wl.sim
geoms = [g for g in sim._geometries()] if hasattr(sim, "_geometries") else None
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
pr.disable()
print("3 steps", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
