"""Run the cfg1 bench workload for a few steps (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = bench.GpuWorkload(bench.make_inputs())
for _ in range(steps):
    wl.step()
torch.cuda.synchronize()
print("ok")
