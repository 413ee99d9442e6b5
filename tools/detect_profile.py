"""Host profile of the cfg3 detection phase (collision.detect_soa)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_06946_b200 import collision  # noqa: E402

wl = bench.Cfg3Workload()
wl.step()
torch.cuda.synchronize()
orig = collision.detect_soa
pr = cProfile.Profile()


def wrapped(*a, **k):
    pr.enable()
    try:
        return orig(*a, **k)
    finally:
        pr.disable()


collision.detect_soa = wrapped
import paper_2306_06946_b200.scene as scm  # noqa: E402

scm.detect_soa = wrapped
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
