"""Proximity update p_a/p_b +=/-= h^2 U_o t (reference constraints.py:238-243)
through cnb_prox_update: the lower-triangle tile path for large objects and the
warp-per-row GEMV for small ones, against a float64 torch product."""

import numpy as np
import pytest
import torch

from paper_2306_06946_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mo,pad,gathered", [(50, 0, False), (333, 1, False), (700, 3, True), (1111, 0, True)])
def test_prox_update_matches_dense_product(mo, pad, gathered):
    rng = np.random.default_rng(mo)
    n = 3 * mo
    B = rng.standard_normal((n, n))
    Ufull = B @ B.T / n                               # symmetric, like U_o = S C S^T
    Ufull = 0.5 * (Ufull + Ufull.T)
    ldu = n + pad                                     # odd leading dimensions too
    U = torch.zeros((n, ldu), dtype=torch.float64, device="cuda")
    U[:, :n] = torch.as_tensor(Ufull, device="cuda")
    m = mo + 17 if gathered else mo
    idx = np.sort(rng.choice(m, mo, replace=False)) if gathered else np.arange(mo)
    side = rng.choice(np.array([1, -1], dtype=np.int8), mo)
    t = torch.as_tensor(rng.standard_normal(3 * m), device="cuda")
    p_a = torch.as_tensor(rng.standard_normal(3 * m), device="cuda")
    p_b = torch.as_tensor(rng.standard_normal(3 * m), device="cuda")
    h = 0.01
    idx_t = torch.as_tensor(idx, device="cuda")
    side_t = torch.as_tensor(side, device="cuda")
    ea, eb = p_a.clone(), p_b.clone()
    pa0, pb0 = p_a.clone(), p_b.clone()
    tg = t.reshape(-1, 3)[idx_t].reshape(-1)
    y = (h * h) * (torch.as_tensor(Ufull, device="cuda") @ tg)
    rows = (3 * idx_t[:, None] + torch.arange(3, device="cuda")).reshape(-1)
    sgn = torch.as_tensor(np.repeat(side, 3), device="cuda")
    ea[rows[sgn > 0]] += y[sgn > 0]
    eb[rows[sgn < 0]] -= y[sgn < 0]
    _lib.call("cnb_prox_update", mo, U.data_ptr(), ldu, idx_t.data_ptr() if gathered else None,
              side_t.data_ptr(), t.data_ptr(), h, p_a.data_ptr(), p_b.data_ptr(), _lib.stream())
    torch.cuda.synchronize()
    scale = float(y.abs().max())
    assert float((p_a - ea).abs().max()) <= 1e-12 * scale + 1e-15
    assert float((p_b - eb).abs().max()) <= 1e-12 * scale + 1e-15
    # repeatable bit for bit (fixed summation order)
    a1, b1 = pa0.clone(), pb0.clone()
    _lib.call("cnb_prox_update", mo, U.data_ptr(), ldu, idx_t.data_ptr() if gathered else None,
              side_t.data_ptr(), t.data_ptr(), h, a1.data_ptr(), b1.data_ptr(), _lib.stream())
    torch.cuda.synchronize()
    assert torch.equal(a1, p_a) and torch.equal(b1, p_b)
