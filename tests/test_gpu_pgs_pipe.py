"""Grid-scale PGS kernels (thousands of groups) against the CPU oracle and each
other.  All three kernels run the reference's Gauss-Seidel iterate
(solver.py:124-202) in the canonical group order; they differ only in the
association of the delta sums, so lambda agrees to rounding (tolerance 1e-9
relative at these condition numbers; the north star asks 1e-6)."""

import numpy as np
import pytest
import torch

import cn_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2306_06946_b200 as m

    return m


def _h(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def rel_err(a, b):
    a, b = _h(a), _h(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _problem(G, seed, rank=48, scale=1.0):
    rng = np.random.default_rng(seed)
    c = 3 * G
    B = rng.standard_normal((c, rank)) / np.sqrt(rank)
    W = scale * (B @ B.T + 0.5 * np.eye(c))
    delta = rng.uniform(-0.02, 0.01, c)
    return W, delta


def _run(cn, monkeypatch, W, delta, cfg, grid, kernel=None):
    monkeypatch.setenv("CNB_PGS_GRID", grid)
    if kernel:
        monkeypatch.setenv("CNB_PGS_KERNEL", kernel)
    else:
        monkeypatch.delenv("CNB_PGS_KERNEL", raising=False)
    return cn.pgs(W, delta, 0.01, cfg)


@pytest.mark.parametrize("G,mu", [(300, 0.4), (140, 0.0), (1000, 0.8)])
def test_pipe_kernel_matches_oracle_fixed_sweeps(cn, monkeypatch, G, mu):
    """Ragged last block (G % 32 != 0), frictionless and sticky cases, fixed budget."""
    W, delta = _problem(G, G)
    sweeps = 12
    lam_o, dend_o, it_o, hist_o, _ = orc.pgs(W, delta, 0.01, sweeps, 1e-300, mu)
    r = _run(cn, monkeypatch, W, delta, cn.PgsConfig(sweeps, 1e-300, mu), "1")
    assert r.iterations == it_o == sweeps
    assert rel_err(r.lam, lam_o) <= 1e-9
    assert rel_err(r.delta_end, dend_o) <= 1e-9
    assert np.allclose(r.eps_history, hist_o, rtol=1e-6, atol=0)


def test_pipe_kernel_convergence_count(cn, monkeypatch):
    """Tolerance-driven stop: same sweep count and epsilon history as the oracle."""
    W, delta = _problem(400, 3)
    lam_o, dend_o, it_o, hist_o, conv_o = orc.pgs(W, delta, 0.01, 300, 1e-7, 0.5)  # 195 sweeps
    r = _run(cn, monkeypatch, W, delta, cn.PgsConfig(300, 1e-7, 0.5), "1")
    assert conv_o and r.converged
    assert r.iterations == it_o
    assert rel_err(r.lam, lam_o) <= 1e-9
    assert np.allclose(r.eps_history, hist_o, rtol=1e-6, atol=0)


def test_grid_kernels_agree_with_single_cta(cn, monkeypatch):
    """3000 groups: pipelined kernel, one-step-lookahead kernel and the single-CTA
    kernel produce the same iterate; the pipelined kernel is bitwise repeatable."""
    W, delta = _problem(3000, 11, rank=64)
    cfg = cn.PgsConfig(15, 1e-300, 0.4)
    r_pipe = _run(cn, monkeypatch, W, delta, cfg, "1")
    lam_pipe = _h(r_pipe.lam).copy()
    r_pipe2 = _run(cn, monkeypatch, W, delta, cfg, "1")
    assert np.array_equal(_h(r_pipe2.lam), lam_pipe)
    r_grid = _run(cn, monkeypatch, W, delta, cfg, "1", kernel="grid")
    r_one = _run(cn, monkeypatch, W, delta, cfg, "0")
    assert rel_err(lam_pipe, r_one.lam) <= 1e-9
    assert rel_err(r_grid.lam, r_one.lam) <= 1e-9
    assert rel_err(r_pipe.delta_end, r_one.delta_end) <= 1e-9
    lam = lam_pipe.reshape(-1, 3)
    assert (lam[:, 0] >= 0).all()
    assert (np.hypot(lam[:, 1], lam[:, 2]) <= 0.4 * lam[:, 0] * (1 + 1e-9) + 1e-12).all()


def test_pipe_kernel_regularises_duplicate_groups(cn, monkeypatch):
    """Two identical groups make W's 6x6 block singular but every 3x3 block
    regular; a rank-deficient diagonal block gets the trace shift (solver.py:99-121)."""
    W, delta = _problem(200, 5)
    W[150:153, :] = W[30:33, :]
    W[:, 150:153] = W[:, 30:33]
    W[153:156, 153:156] = np.outer([1.0, 2.0, 3.0], [1.0, 2.0, 3.0]) * 1e-3  # singular diagonal block
    W[153:156, :153] = 0.0
    W[:153, 153:156] = 0.0
    W[153:156, 156:] = 0.0
    W[156:, 153:156] = 0.0
    lam_o, dend_o, it_o, _, _ = orc.pgs(W, delta, 0.01, 10, 1e-300, 0.0)
    r = _run(cn, monkeypatch, W, delta, cn.PgsConfig(10, 1e-300, 0.0), "1")
    assert r.iterations == it_o
    assert rel_err(r.lam, lam_o) <= 1e-9
    assert rel_err(r.delta_end, dend_o) <= 1e-9


def test_pipe_kernel_singular_block_raises(cn, monkeypatch):
    W, delta = _problem(300, 9)
    W[3 * 170, 3 * 170] = -1.0  # W_nn <= 0 in block 5
    monkeypatch.setenv("CNB_PGS_GRID", "1")
    with pytest.raises(cn.SingularBlockError):
        cn.pgs(W, delta, 0.01, cn.PgsConfig(5, 1e-300, 0.4))
