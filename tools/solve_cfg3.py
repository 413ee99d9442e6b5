"""Single-RHS solve time on one cfg3 body's factor (225k DoF, corotational
5-tet grid), CUDA events; algorithmic bytes 2 x 8 nnz(L) per solve."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_06946_b200 as cn  # noqa: E402

mesh = cn.five_tet_grid((50, 30, 50), 0.01)
body = cn.SoftBody(mesh, young=1e4, poisson=0.4, density=1000.0, material="corotational")
A, b = body.assemble(body.initial_state(), 0.01, (0.0, -9.81, 0.0))
F = cn.Factorization(A)
rhs = torch.randn(body.n_dofs, dtype=torch.float64, device="cuda")
x = torch.empty_like(rhs)
for _ in range(3):
    F.solve_device(rhs.reshape(1, -1), out=x.reshape(1, -1))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    F.solve_device(rhs.reshape(1, -1), out=x.reshape(1, -1))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"dofs": body.n_dofs, "nnz_L": F.nnz_L, "solve_ms": round(ms, 3),
                  "gbs": round(16.0 * F.nnz_L / (ms * 1e-3) / 1e9, 1)}))
import ctypes  # noqa: E402

from paper_2306_06946_b200 import _lib  # noqa: E402

prof = (ctypes.c_double * 64)()
F.solve_device(rhs.reshape(1, -1), out=x.reshape(1, -1))
torch.cuda.synchronize()
_lib.call("cnb_solve_profile", prof)
ts = [prof[k] for k in range(64) if prof[k] > 0]
print(json.dumps({"phase_us": [round((b - a) / 1e3, 1) for a, b in zip(ts, ts[1:])], "levels": F.n_levels}))
