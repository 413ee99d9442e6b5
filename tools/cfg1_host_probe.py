"""cfg1 step: host time of each phase call (no sync) against its device time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402


def main():
    wl = bench.GpuWorkload(workloads.cfg1_inputs())
    for _ in range(3):
        wl.step()
    torch.cuda.synchronize()
    cn = wl.cn
    rows = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A, _ = wl.body.assemble(wl.state, bench.H, (0.0, -9.81, 0.0))
        t1 = time.perf_counter()
        wl.F.refactor_async(A.values)
        t2 = time.perf_counter()
        wl.wg = cn.assemble_Wg({0: wl.S}, {0: wl.F})
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        rows.append({"host_assemble_ms": round((t1 - t0) * 1e3, 3), "host_refactor_ms": round((t2 - t1) * 1e3, 3),
                     "host_wg_ms": round((t3 - t2) * 1e3, 3), "wait_after_ms": round((t4 - t3) * 1e3, 3)})
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
