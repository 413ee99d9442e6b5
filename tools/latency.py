"""Dependent-op latencies on the GPU (cycles/op) and the DMMA throughput peak."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2306_06946_b200 import _lib  # noqa: E402

out = (ctypes.c_double * 12)()
_lib.call("cnb_bench_latency", out, _lib.stream())
dm = (ctypes.c_double * 1)()
_lib.call("cnb_bench_dmma", 4096, dm, _lib.stream())
names = ["dfma", "dadd", "ddiv", "dsqrt", "shfl64_plus_dadd", "ffma", "dsel_plus_dadd", "rsq64h_plus_dadd", "dmul"]
thr = ["dfma_issue", "lds64_broadcast_issue", "potrf_bulk_step"]
print(json.dumps({"cycles_per_dependent_op": dict(zip(names, [round(v, 2) for v in out[:9]])),
                  "single_warp_cycles": dict(zip(thr, [round(v, 2) for v in out[9:]])),
                  "dmma_tflops": round(dm[0], 2), "gpu": torch.cuda.get_device_name(0)}))
