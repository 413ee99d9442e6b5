"""Per-block time of the pipelined PGS kernel against the group count G on a
synthetic dense SPD Delassus operator (fixed 10-sweep budget): flat per-block
time = bound by the sequential chain; time growing with G = bound by the
helpers' streaming of W."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_06946_b200 as cn  # noqa: E402
from paper_2306_06946_b200 import _device as dv  # noqa: E402
from paper_2306_06946_b200.solver import pgs_device  # noqa: E402

for G in [int(x) for x in (sys.argv[1:] or ["1500", "3000", "5000", "7301"])]:
    c = 3 * G
    g = torch.Generator(device="cuda").manual_seed(1)
    B = torch.randn(c, 64, device="cuda", dtype=torch.float64, generator=g) / 8.0
    W = dv.square(c)
    torch.matmul(B, B.T, out=W)
    W.diagonal().add_(1.0)
    delta = torch.randn(c, device="cuda", dtype=torch.float64, generator=g) * 1e-3
    delta.view(-1, 3)[:, 0] -= 2e-3
    cfg = cn.PgsConfig(10, 1e-300, 0.4)
    pgs_device(W, delta, 0.01, cfg)
    torch.cuda.synchronize()
    if os.environ.get("CNB_PGS_PROFILE") == "1":  # reset the phase sums after the warm-up
        import ctypes
        from paper_2306_06946_b200 import _lib
        _lib.lib().cnb_pgs_profile((ctypes.c_double * 32)())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = pgs_device(W, delta, 0.01, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nb = (G + 25) // 26
    import ctypes
    from paper_2306_06946_b200 import _lib
    prof = (ctypes.c_double * 32)()
    if os.environ.get("CNB_PGS_PROFILE") == "1" and _lib.lib().cnb_pgs_profile(prof) == 0:
        print(json.dumps({"groups": G, "us_per_block_step": {k: round(prof[k] / (res.iterations * nb) / 1965.0, 3)
                                                             for k in range(32) if prof[k]}}), flush=True)
    print(json.dumps({"groups": G, "sweeps": res.iterations, "ms_per_sweep": round(ms / res.iterations, 4),
                      "us_per_block": round(ms * 1e3 / res.iterations / nb, 3),
                      "w_gbs": round(8.0 * c * c / (ms / res.iterations * 1e-3) / 1e9, 1)}), flush=True)
    del W, B
