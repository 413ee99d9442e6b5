"""Numeric factorisation of one cfg3 body (50x30x50-node corotational 5-tet grid,
225k DoF): ms and TFLOP/s per refactor (CUDA events), for ncu launch lists.

    python tools/factor_profile.py --reps 3
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=[50, 30, 50])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2306_06946_b200 as cn

    mesh = cn.five_tet_grid(tuple(args.shape), 0.01)
    body = cn.SoftBody(mesh, young=1e4, poisson=0.4, density=1000.0, material="corotational")
    state = body.initial_state()
    A, _ = body.assemble(state, 0.01, (0.0, -9.81, 0.0))
    F = cn.Factorization(A)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.refactor_async(A.values)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    F.check_status()
    import ctypes

    from paper_2306_06946_b200 import _lib

    pp = (ctypes.c_double * 8)()
    _lib.call("cnb_potrf_profile", pp)
    n = max(pp[7], 1)
    print(json.dumps({"potrf_cycles_per_launch": {k: round(pp[i] / n) for i, k in enumerate(
        ["loads", "elimination_loop"])}, "launches": pp[7]}), flush=True)
    ms = min(times)
    print(json.dumps({"dofs": body.n_dofs, "supernodes": F.n_supernodes, "levels": F.n_levels, "nnz_L": F.nnz_L,
                      "gflop": round(F.flops / 1e9, 1), "ms": round(ms, 3),
                      "tflops": round(F.flops / (ms * 1e-3) / 1e12, 2)}), flush=True)


if __name__ == "__main__":
    main()
