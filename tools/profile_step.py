"""Run the default bench workload (cfg3 Simulation.step) for a few steps, for ncu
launch lists and captures:  python tools/profile_step.py [steps] [cfg3|cfg1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
which = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
import workloads  # noqa: E402

wl = bench.Cfg3Workload() if which == "cfg3" else bench.GpuWorkload(workloads.cfg1_inputs())
for _ in range(steps):
    wl.step()
torch.cuda.synchronize()
print("ok")
