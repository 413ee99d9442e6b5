"""cfg4 step-time jitter probe: per-step device time (CUDA events), host time and
caching-allocator activity over a run of steps after the bench's pre-roll."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    wl = bench.Cfg4Workload(0, 1)
    for _ in range(bench.CFG4_PREROLL):
        wl.step()
    torch.cuda.synchronize()
    rows = []
    for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
        s0 = torch.cuda.memory_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        pairs = wl.step()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        s1 = torch.cuda.memory_stats()
        rows.append({"step": i, "dev_ms": round(e0.elapsed_time(e1), 2), "host_ms": round((t1 - t0) * 1e3, 2),
                     "pairs": pairs,
                     "segments_new": s1["segment.all.allocated"] - s0["segment.all.allocated"],
                     "segments_freed": s1["segment.all.freed"] - s0["segment.all.freed"],
                     "alloc_retries": s1["num_alloc_retries"] - s0["num_alloc_retries"]})
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
