"""cfg3 probe: step the benched two-block scene and print per-step pairs, sweeps,
device memory and wall time (steady-state behaviour of the bench workload)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06946_b200 as cn  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
shift = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
gap = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
sim = cn.Simulation(bench.make_cfg3_config(cn, shift=shift, gap=gap))
for s in range(steps):
    t0 = time.perf_counter()
    try:
        rep = sim.step()
    except Exception as exc:
        print("step", s, "failed:", exc, flush=True)
        print(torch.cuda.memory_summary(abbreviated=True), flush=True)
        raise
    torch.cuda.synchronize()
    print(f"step {s} pairs {rep.c_groups} newton {rep.newton_iterations} sweeps {rep.pgs_iterations_total} "
          f"pen_after {rep.pen_after:.3e} wall {1e3 * (time.perf_counter() - t0):.1f} ms "
          f"alloc {torch.cuda.memory_allocated() / 2**30:.1f} GiB reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB "
          f"free {torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB", flush=True)
