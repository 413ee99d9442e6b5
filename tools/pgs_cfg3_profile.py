"""PGS on the benched cfg3 Delassus operators: W = D W_g D^T of the first
Newton iteration at step 0 and at step 2 (sliding), fixed sweep budget, with
the pipe kernel's phase profile (CNB_PGS_PROFILE=1)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_06946_b200 as cn  # noqa: E402
from paper_2306_06946_b200 import _lib  # noqa: E402
from paper_2306_06946_b200.solver import pgs_device  # noqa: E402

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sim = cn.Simulation(bench.make_cfg3_config(cn, shift=bench.CFG3_SHIFT, gap=bench.CFG3_GAP))
for step in range(3):
    if step in (0, 2):
        ctx = sim.prepare_step(build_wg=True)[0]
        D = cn.assemble_direction(ctx.detection_frames)
        W = cn.rebuild_W_fast(D, ctx.wg).W
        delta = cn.compute_violation(D, ctx.p_a0, ctx.p_b0).delta
        cfgs = {"fixed": cn.PgsConfig(sweeps, 1e-300, 0.4), "tol": cn.PgsConfig(30, 1e-6, 0.4),
                "nofric": cn.PgsConfig(sweeps, 1e-300, 0.0)}
        for name, cfg in cfgs.items():
            pgs_device(W, delta, 0.01, cfg)
            torch.cuda.synchronize()
            prof = (ctypes.c_double * 32)()
            have = _lib.lib().cnb_pgs_profile(prof) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = pgs_device(W, delta, 0.01, cfg)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            G = W.shape[0] // 3
            lam = res.lam.reshape(-1, 3)
            out = {"step": step, "cfg": name, "groups": G, "sweeps": res.iterations, "ms": round(ms, 3),
                   "ms_per_sweep": round(ms / res.iterations, 4),
                   "active": int((lam[:, 0] > 0).sum()), "sliding": int(
                       ((lam[:, 1] ** 2 + lam[:, 2] ** 2).sqrt() >= 0.4 * lam[:, 0] * (1 - 1e-9)).logical_and(
                           lam[:, 0] > 0).sum())}
            if have:
                _lib.lib().cnb_pgs_profile(prof)
                nb = (G + 25) // 26
                out["us_per_block_step"] = {k: round(prof[k] / (res.iterations * nb) / 1965.0, 3)
                                            for k in range(32) if prof[k]}
            print(json.dumps(out), flush=True)
        del W
    sim.step()
