"""Host-side profile of one cfg3 Simulation.step (cProfile, cumulative)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

wl = bench.Cfg3Workload()
for _ in range(2):
    wl.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
wl.step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
