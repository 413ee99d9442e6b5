"""Single-RHS solve latency on the cfg1 factor (CUDA events), and the cfg1
Newton iteration's parts: rebuild W, apply D^T, S^T t, solve."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_06946_b200 import _lib  # noqa: E402


def timed(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


import workloads  # noqa: E402

wl = bench.GpuWorkload(workloads.cfg1_inputs())
wl.step()
torch.cuda.synchronize()
m = bench.N_CONTACTS
D = wl.Ds[0]
st = _lib.stream()
out = {
    "rebuild_w_us": timed(lambda: _lib.call("cnb_rebuild_w", m, D.data_ptr(), wl.wg.wg.data_ptr(), 3 * m,
                                            wl.W.data_ptr(), 3 * m, st)),
    "apply_dt_us": timed(lambda: _lib.call("cnb_apply_dt", m, D.data_ptr(), wl.lams[0].data_ptr(),
                                           wl.t.data_ptr(), None, st)),
    "st_t_us": timed(lambda: wl.S.rmatvec(wl.t, out=wl.rhs, alpha=bench.H)),
    "solve_us": timed(lambda: wl.F.solve_device(wl.rhs.reshape(1, -1), out=wl.dx[0].reshape(1, -1))),
}
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
import ctypes  # noqa: E402

prof = (ctypes.c_double * 64)()
wl.F.solve_device(wl.rhs.reshape(1, -1), out=wl.dx[0].reshape(1, -1))
torch.cuda.synchronize()
_lib.call("cnb_solve_profile", prof)
ts = [prof[k] for k in range(64) if prof[k] > 0]
print(json.dumps({"phase_us": [round((b - a) / 1e3, 2) for a, b in zip(ts, ts[1:])], "levels": wl.F.n_levels}))
