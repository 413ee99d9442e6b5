"""cfg4 profile: per-phase device time of one batched step, PGS sweep statistics
per Newton iteration, and the batched PGS kernel's per-sweep time vs the number
of copies in the launch (fixed sweep count)."""

import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2306_06946_b200 import _lib  # noqa: E402


def main():
    wl = bench.Cfg4Workload(0, 1)
    B = wl.B
    for _ in range(bench.CFG4_PREROLL):
        B.step()
    B.check()
    # record per-iteration sweep counts via a wrapper
    orig = _lib.call
    log = []

    def call(name, *a):
        if name == "cnb_pgs_batched":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = orig(name, *a)
            e1.record()
            ic_ptr = a[13]
            log.append((e0, e1, ic_ptr))
            return r
        return orig(name, *a)

    _lib.call = call
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    B.step()
    ev[1].record()
    _lib.call = orig
    torch.cuda.synchronize()
    out = {"step_ms": ev[0].elapsed_time(ev[1]), "pgs_ms": [a.elapsed_time(b) for a, b, _ in log]}
    it = B.last["iters"].cpu().numpy()
    cnt = B.last["pairs"]["cnt"]
    out["last_iter_sweeps"] = dict(max=int(it[:, 0].max()), mean=float(it[:, 0].mean()),
                                   p99=float(np.percentile(it[:, 0], 99)), conv=int(it[:, 1].sum()))
    out["sweeps_per_iteration"] = [dict(max=int(x[:, 0].max()), mean=round(float(x[:, 0].mean()), 1),
                                        p90=float(np.percentile(x[:, 0], 90)), unconverged=int((x[:, 1] == 0).sum()))
                                   for x in (t.cpu().numpy() for t in B.last["iters_all"])]
    out["groups"] = dict(max=int(cnt.max()), mean=float(cnt.mean()), min=int(cnt.min()))
    # fixed-sweep timing of the batched kernel vs copies in the launch
    P = B.last["pairs"]
    ns = B.ns
    m = P["m"]
    c_tot = 3 * m
    W = torch.empty(P["wsize"], dtype=torch.float64, device="cuda")
    Wg = torch.empty_like(W)
    _lib.call("cnb_batch_wg_gather", ns, int(P["boff_h"][-1]), P["boff"].data_ptr(), P["poff"].data_ptr(),
              P["woff"].data_ptr(), P["cand"].data_ptr(), B.vids.data_ptr(), B.Ainv.data_ptr(), B.n, Wg.data_ptr(),
              _lib.stream())
    _lib.call("cnb_batch_rebuild_w", ns, int(P["boff_h"][-1]), P["boff"].data_ptr(), P["poff"].data_ptr(),
              P["woff"].data_ptr(), B.last["frames"].data_ptr(), Wg.data_ptr(), W.data_ptr(), _lib.stream())
    delta = torch.full((c_tot,), -1e-4, dtype=torch.float64, device="cuda")
    lam, dend = torch.empty_like(delta), torch.empty_like(delta)
    SW = 50
    eps = torch.empty((ns, SW), dtype=torch.float64, device="cuda")
    ic = torch.zeros((ns, 2), dtype=torch.int32, device="cuda")
    st = _lib.status(torch.device("cuda"))
    timing = {}
    exp = os.environ.pop("BATCH_EXP", None)
    if exp:
        os.environ["CNB_PGS_COPY_EXP"] = exp
    for k in (1, 2, 148, 296, 592, 1024):
        k = min(k, ns)
        g_off = np.ascontiguousarray(P["poff_h"][:k + 1])
        w_off = np.ascontiguousarray(P["woff_h"][:k])
        mus = np.ascontiguousarray(B.mus[:k])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(2):
            e0.record()
            _lib.call("cnb_pgs_batched", k, g_off.ctypes.data, w_off.ctypes.data, mus.ctypes.data, W.data_ptr(),
                      delta.data_ptr(), B.h, 0.0, SW, lam.data_ptr(), dend.data_ptr(), eps.data_ptr(), ic.data_ptr(), None,
                      st.ptr, _lib.stream())
            e1.record()
        torch.cuda.synchronize()
        timing[k] = round(e0.elapsed_time(e1) * 1e3 / SW, 2)
    os.environ.pop("CNB_PGS_COPY_EXP", None)
    out["us_per_sweep_fixed50_by_copies"] = timing
    if os.environ.get("CNB_PGS_PROFILE") == "1":
        buf = (ctypes.c_double * 32)()
        _lib.lib().cnb_pgs_profile(buf)  # reset
        g_off = np.ascontiguousarray(P["poff_h"][:2])
        w_off = np.ascontiguousarray(P["woff_h"][:1])
        mus = np.ascontiguousarray(B.mus[:1])
        _lib.call("cnb_pgs_batched", 1, g_off.ctypes.data, w_off.ctypes.data, mus.ctypes.data, W.data_ptr(),
                  delta.data_ptr(), B.h, 0.0, SW, lam.data_ptr(), dend.data_ptr(), eps.data_ptr(), ic.data_ptr(), None,
                  st.ptr, _lib.stream())
        torch.cuda.synchronize()
        _lib.check(_lib.lib().cnb_pgs_profile(buf), "profile")
        nblk = max(buf[13], 1)
        out["copy_kernel_cycles_per_block"] = {k: round(buf[8 + i] / nblk, 1) for i, k in enumerate(
            ["solve", "solver_wait", "helper_products", "helper_tile_wait", "delta_phase", "blocks",
             "helper_after_stage", "helper_after_loop"])}
        out["blocks"] = buf[13]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
