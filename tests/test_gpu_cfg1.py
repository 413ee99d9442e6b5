"""BASELINE cfg1 (isolated compliance-update bench, 12 000 DoF, 500 barycentric
contacts, 10 frame re-draws) through the benched GPU path against the
reference's own run of the same inputs (tests/golden/cfg1_parity.npz, written
by tests/golden/make_golden.py cfg1_parity with the reference package).

North-star tolerances: W and dx within 1e-9 relative; the S pattern bit-exact.
W_g is compared on 32 sampled rows and through W_g r for a fixed random r (every
entry enters), each W_k on 8 rows and through W_k r, dx_k in full for k = 0, 4, 9
and on 600 sampled DoFs for every k."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _h(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _rel(a, b):
    return np.abs(_h(a) - b).max() / np.abs(b).max()


@pytest.fixture(scope="module")
def run():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench

    wl = bench.GpuWorkload(bench.make_inputs())
    Ws = []
    # the benched step, with each re-draw's W kept for the comparison
    orig = wl._lib.call

    def spy(name, *a):
        r = orig(name, *a)
        if name == "cnb_rebuild_w":
            Ws.append(wl.W.clone())
        return r

    wl._lib.call = spy
    try:
        dx = wl.step().clone()
    finally:
        wl._lib.call = orig
    return wl, dx, Ws


def test_signed_mapping_pattern(run, golden):
    g = golden("cfg1_parity.npz")
    S = run[0].S.csr
    assert np.array_equal(S.indptr, g["S_indptr"])
    assert np.array_equal(S.indices, g["S_indices"])
    assert np.array_equal(S.data, g["S_data"])


def test_mapping_compliance(run, golden):
    g = golden("cfg1_parity.npz")
    wg = _h(run[0].wg.wg)
    assert _rel(wg[g["rows"]], g["wg_rows"]) <= 1e-9
    assert _rel(wg @ g["r"], g["wg_r"]) <= 1e-9


def test_rebuilt_delassus_and_corrections(run, golden):
    g = golden("cfg1_parity.npz")
    wl, dx, Ws = run
    assert len(Ws) == 10
    for k in range(10):
        W = _h(Ws[k])
        assert _rel(W[g["rows"][:8]], g[f"W{k}_rows"]) <= 1e-9, k
        assert _rel(W @ g["r"], g[f"W{k}_r"]) <= 1e-9, k
        d = _h(dx[k])
        assert _rel(d[g["dsel"]], g[f"dx{k}_sel"]) <= 1e-9, k
        if f"dx{k}" in g:
            assert _rel(d, g[f"dx{k}"]) <= 1e-9, k
