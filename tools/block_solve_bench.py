"""Cycles per group of the PGS warp block solve, per variant (diagnostic)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2306_06946_b200 import _lib  # noqa: E402

torch.cuda.init()
out = (ctypes.c_double * 2)()
res = {}
names = ["fma-update", "h2-prescaled", "branchless-rsqrt", "both",
         "proj:fma-update", "proj:h2-prescaled", "proj:branchless-rsqrt", "proj:both", "v2", "proj:v2", "v3", "proj:v3", "v4", "proj:v4", "proj:v5-26x78-next-block", "proj:v4-26x78"]
for v, name in enumerate(names):
    _lib.call("cnb_bench_block_solve", v, 50, out, _lib.stream())
    _lib.call("cnb_bench_block_solve", v, 2000, out, _lib.stream())
    res[name] = round(out[0], 1)
print(json.dumps({"cycles_per_group": res}))
cont = {}
for mode, name in enumerate(["idle", "lds", "shfl", "global-poll", "bulk-copy", "dfma"]):
    _lib.call("cnb_bench_contention", mode, 50, out, _lib.stream())
    _lib.call("cnb_bench_contention", mode, 2000, out, _lib.stream())
    cont[name] = round(out[0], 1)
print(json.dumps({"cycles_per_group_under_load": cont}))
