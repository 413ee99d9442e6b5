"""Grid PGS phase profile: random SPD-ish W of G groups, fixed sweep budget.

    CNB_PGS_PROFILE=1 python tools/pgs_profile.py --groups 8000 --sweeps 30
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, nargs="+", default=[2000, 8000])
    ap.add_argument("--sweeps", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2306_06946_b200 as cn
    from paper_2306_06946_b200 import _lib
    from paper_2306_06946_b200.solver import pgs_device

    for G in args.groups:
        c = 3 * G
        g = torch.Generator(device="cuda").manual_seed(G)
        R = torch.randn((c, c), dtype=torch.float64, device="cuda", generator=g)
        W = (R + R.T) * (0.2 / c ** 0.5)
        W.diagonal().add_(4.0)
        del R
        delta = -torch.rand(c, dtype=torch.float64, device="cuda", generator=g) * 1e-3
        cfg = cn.PgsConfig(args.sweeps, 1e-300, 0.4)
        pgs_device(W, delta, 0.01, cfg)  # warm-up
        torch.cuda.synchronize()
        prof = (ctypes.c_double * 32)()
        have_prof = _lib.lib().cnb_pgs_profile(prof) == 0
        times = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = pgs_device(W, delta, 0.01, cfg)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        sweeps = res.iterations
        nb = (G + 31) // 32 if os.environ.get("CNB_PGS_KERNEL", "pipe").startswith("g") else (G + 25) // 26
        out = {"groups": G, "sweeps": sweeps, "ms": round(min(times), 3),
               "ms_per_sweep": round(min(times) / sweeps, 4),
               "us_per_block_step": round(min(times) * 1e3 / (sweeps * nb), 3),
               "hbm_roofline_ms_per_sweep": round(8.0 * c * c / 6545.6e9 * 1e3, 4)}
        if have_prof:
            _lib.lib().cnb_pgs_profile(prof)
            steps = args.reps * sweeps * nb
            names = [str(k) for k in range(32)]
            # pipe kernel slots are SM cycles (clock64); microseconds at the 1965 MHz clock
            out["us_per_step"] = {n: round(prof[k] / steps / 1965.0, 3) for k, n in enumerate(names) if prof[k]}
        print(json.dumps(out), flush=True)
        del W


if __name__ == "__main__":
    main()
