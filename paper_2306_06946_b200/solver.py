"""Projected Gauss-Seidel and the recursive corrective-motion schemes on the GPU.

Mirrors /root/reference/pkg/src/contactnewton/solver.py: ``PgsConfig`` /
``NewtonConfig`` (52-79), ``regularize`` (99-121), ``local_solve`` (124-165),
``pgs`` (168-202), ``StepContext`` / ``CorrectionResult`` (208-242),
``newton_standard`` (260-311), ``newton_fast`` (314-367).

``newton_fast`` keeps the whole loop on the device: re-linearisation, the
W rebuild, the violation, PGS, the proximity update and the impulse
accumulation are kernels on one stream; the host only reads a scalar when an
early exit is enabled (non-negative tolerance).  Per-phase wall times are
taken with CUDA events and resolved once at the end.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .collision import PairTable, frames_tensor, relinearize_device
from .constraints import (
    DirectionMatrix,
    MappingDelassus,
    assemble_direction,
    compute_violation,
    prox_update_inplace,
    rebuild_W_fast,
)
from .errors import DimensionMismatchError, SingularBlockError, ValidationError

SCHEMES = ("single", "standard", "fast")


ORDERINGS = ("exact", "coloured")


@dataclass
class PgsConfig:
    """PGS budget and friction (solver.py:52-64).  ``ordering`` (not in the
    reference) selects the group order: "exact" — the reference's canonical
    Gauss-Seidel order (default, parity-pinned); "coloured" — groups coloured
    so that no two groups sharing a DoF share a colour, each colour updated at
    once (the north star's graph-coloured variant; a different iterate, checked
    on the converged lambda only)."""

    max_iterations: int = 30
    tolerance: float = 1e-6
    friction: float = 0.5
    ordering: str = "exact"
    relaxation: float = 1.0  # coloured ordering only: under-relaxation of each group's change

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValidationError("pgs.max_iterations must be >= 1")
        if self.tolerance <= 0:
            raise ValidationError("pgs.tolerance must be positive")
        if self.friction < 0:
            raise ValidationError("friction coefficient must be >= 0")
        if self.ordering not in ORDERINGS:
            raise ValidationError(f"unknown pgs ordering {self.ordering!r}, pick from {ORDERINGS}")
        if not 0.0 < self.relaxation <= 1.0:
            raise ValidationError("pgs.relaxation must be in (0, 1]")


@dataclass
class NewtonConfig:
    scheme: str = "single"
    max_iterations: int = 5
    penetration_tol: float = 1e-5
    relinearize: bool = True
    rotation_tol: float = 1e-4

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValidationError(f"unknown scheme {self.scheme!r}, pick from {SCHEMES}")
        if self.max_iterations < 1:
            raise ValidationError("newton.max_iterations must be >= 1")


class PgsResult:
    """lam, delta_end (device); iterations / eps_history / converged read lazily."""

    def __init__(self, lam, delta_end, eps_buf, ic_buf, status=None):
        self.lam = lam
        self.delta_end = delta_end
        self._eps = eps_buf
        self._ic = ic_buf
        self._status = status
        self._host = None

    def _resolve(self):
        if self._host is None:
            if self._status is not None:
                self._status.raise_if_set("pgs")
            if self._ic is None:
                self._host = (0, [], True)
            else:
                ic = self._ic.cpu().numpy()
                it = int(ic[0])
                self._host = (it, [float(x) for x in self._eps[:it].cpu().numpy()], bool(ic[1]))
        return self._host

    @property
    def iterations(self) -> int:
        return self._resolve()[0]

    @property
    def eps_history(self) -> list:
        return self._resolve()[1]

    @property
    def converged(self) -> bool:
        return self._resolve()[2]


@dataclass
class LambdaState:
    lam: torch.Tensor
    accumulated: torch.Tensor


def regularize(W):
    """Shift (numerically) singular 3x3 diagonal blocks by 1e-10 trace(W)/c
    (solver.py:99-121).  The PGS kernel applies the same rule internally;
    this standalone form exists for API parity."""
    W = dv.f64(W)
    c = W.shape[0]
    if c == 0:
        return W
    shift = 1e-10 * float(torch.trace(W)) / c
    if shift <= 0:
        shift = 1e-30
    g = c // 3
    blocks = W.reshape(g, 3, g, 3).diagonal(dim1=0, dim2=2).permute(2, 0, 1)
    sym = 0.5 * (blocks + blocks.transpose(1, 2))
    eigs = torch.linalg.eigvalsh(sym)
    scale = torch.clamp(eigs.abs().max(dim=1).values, min=1e-300)
    bad = eigs.min(dim=1).values <= 1e-12 * scale
    if not bool(bad.any()):
        return W
    out = W.clone()
    for gi in torch.nonzero(bad).flatten().tolist():
        out[3 * gi:3 * gi + 3, 3 * gi:3 * gi + 3] += shift * torch.eye(3, dtype=W.dtype, device=W.device)
    return out


def local_solve(alpha: int, W, delta_cur, lam, mu: float, h2: float):
    """One group's Signorini/Coulomb block solve (solver.py:124-165), on the device."""
    W_t, d_t, l_t = dv.mat64(W), dv.f64(delta_cur), dv.f64(lam)
    out = dv.empty(3)
    st = _lib.status(out.device)
    _lib.call("cnb_local_solve", int(alpha), W_t.shape[0] // 3, W_t.data_ptr(), dv.ld(W_t), d_t.data_ptr(),
              l_t.data_ptr(), float(mu), float(h2), out.data_ptr(), st.ptr, _lib.stream())
    st.raise_if_set("local_solve")
    return out


class PgsWorkspace:
    """Reusable device buffers for one PGS call site (no per-call allocation)."""

    def __init__(self, c: int, max_iter: int):
        self.c = c
        self.lam = dv.empty(c)
        self.delta_end = dv.empty(c)
        self.eps = dv.empty(max(1, max_iter))
        self.ic = dv.zeros(2, dtype=torch.int32)
        self.shift = dv.empty(max(1, c // 3))


def colour_groups(S_by_object: dict, groups: int):
    """Greedy colouring of the contact groups in canonical order: two groups that
    share a DoF column of any object's S (the sparsified coupling graph of W)
    get different colours.  Returns (colour_ptr, groups by colour), int64; the
    groups of a colour stay in canonical order."""
    keys = [[] for _ in range(groups)]
    for oid, S in sorted(S_by_object.items()):
        csr = S.sorted_csr if hasattr(S, "sorted_csr") else S.tocsr()
        rows = np.repeat(np.arange(csr.shape[0]), np.diff(csr.indptr))
        for i, k in zip(rows // 3, csr.indices // 3):  # (group, node of this object)
            keys[i].append((oid, int(k)))
    colour = np.empty(groups, dtype=np.int64)
    used: dict = {}
    for i in range(groups):
        taken = set()
        for k in set(keys[i]):
            taken |= used.get(k, set())
        col = 0
        while col in taken:
            col += 1
        colour[i] = col
        for k in set(keys[i]):
            used.setdefault(k, set()).add(col)
    order = np.lexsort((np.arange(groups), colour)).astype(np.int64)
    ptr = np.zeros(int(colour.max(initial=-1)) + 2, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(colour, minlength=len(ptr) - 1))
    return ptr, order


def pgs_device(W: torch.Tensor, delta_base: torch.Tensor, h: float, config: PgsConfig,
               ws: PgsWorkspace | None = None, delta_end: bool = True, colours=None) -> PgsResult:
    """Asynchronous PGS: launches and returns device results (no host sync).
    ``delta_end=False`` skips the final pass over W (the caller forms delta_end
    another way) and records the regularisation shifts in ``ws.shift``.
    ``config.ordering == "coloured"`` needs ``colours`` = colour_groups(...)."""
    c = int(delta_base.shape[0])
    dev = delta_base.device
    if c == 0:
        return PgsResult(dv.zeros(0), dv.zeros(0), None, None)
    if tuple(W.shape) != (c, c):
        raise SingularBlockError(f"W is {tuple(W.shape)}, violation has {c} rows")
    ws = ws or PgsWorkspace(c, config.max_iterations)
    st = _lib.status(dev)
    common = (ws.lam.data_ptr(), ws.delta_end.data_ptr() if delta_end else None, ws.eps.data_ptr(),
              ws.ic.data_ptr(), None if delta_end else ws.shift.data_ptr(), st.ptr, _lib.stream())
    if config.ordering == "coloured":
        if colours is None:
            raise ValidationError("coloured PGS needs the group colouring (solver.colour_groups)")
        ptr, grp = (np.ascontiguousarray(x, dtype=np.int64) for x in colours)
        if len(grp) != c // 3:
            raise DimensionMismatchError(f"colouring covers {len(grp)} groups, W has {c // 3}")
        _lib.call("cnb_pgs_coloured", c // 3, W.data_ptr(), dv.ld(W), delta_base.data_ptr(), float(h),
                  float(config.friction), float(config.tolerance), int(config.max_iterations), ptr.ctypes.data,
                  grp.ctypes.data, len(ptr) - 1, float(config.relaxation), *common)
    else:
        _lib.call("cnb_pgs", c // 3, W.data_ptr(), dv.ld(W), delta_base.data_ptr(), float(h),
                  float(config.friction), float(config.tolerance), int(config.max_iterations), *common)
    return PgsResult(ws.lam, ws.delta_end, ws.eps, ws.ic, st)


def pgs(W, delta_base, h: float, config: PgsConfig, colours=None) -> PgsResult:
    """Sweep the groups until the relative lambda change drops below tolerance
    (solver.py:168-202).  Returns device lam and delta_end."""
    W_t, d_t = dv.mat64(W), dv.f64(delta_base)
    res = pgs_device(W_t, d_t, h, config, colours=colours)
    res._resolve()
    return res


# --- recursive correction ------------------------------------------------------


@dataclass
class StepContext:
    pairs: list
    detection_frames: object
    S_by_object: dict
    F_by_object: dict
    p_a0: torch.Tensor
    p_b0: torch.Tensor
    h: float
    refresh: Callable | None = None
    wg: MappingDelassus | None = None
    table: PairTable | None = None
    colours: tuple | None = None  # coloured PGS: (colour_ptr, groups), built on first use

    def colouring(self):
        if self.colours is None:
            self.colours = colour_groups(self.S_by_object, len(self.pairs))
        return self.colours


@dataclass
class IterationStats:
    rebuild_time: float
    pgs_time: float
    correction_time: float
    pgs_iterations: int
    pgs_eps: float
    penetration: float
    rotation: float


@dataclass
class CorrectionResult:
    dv_by_object: dict
    lam_history: list
    state: LambdaState
    iterations: list = field(default_factory=list)
    final_frames: object = None
    build_wg_time: float = 0.0
    final_correction_time: float = 0.0


def _penetration_device(delta_end: torch.Tensor) -> torch.Tensor:
    if delta_end.numel() == 0:
        return dv.zeros(1)
    return torch.clamp(-delta_end.reshape(-1, 3)[:, 0].min(), min=0.0).reshape(1)


def mechanical_correction(ctx: StepContext, t: torch.Tensor) -> dict:
    """dv_o = h A_o^-1 S_o^T t, one solve per object (solver.py:250-257)."""
    out = {}
    for oid in sorted(ctx.S_by_object):
        S = ctx.S_by_object[oid]
        F = ctx.F_by_object[oid]
        rhs = S.rmatvec(t)
        F.solve_count += 1
        x = F.solve_device(rhs.reshape(1, -1)).reshape(-1)
        out[oid] = x.mul_(ctx.h)
    return out


class _Timer:
    """Phase stamps as CUDA events on the current stream, resolved at the end."""

    def __init__(self):
        self.events = []

    def mark(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.append(e)
        return len(self.events) - 1

    def secs(self, a, b):
        return self.events[a].elapsed_time(self.events[b]) * 1e-3


def newton_fast(ctx: StepContext, ncfg: NewtonConfig, pcfg: PgsConfig) -> CorrectionResult:
    """Fast recursive correction (paper Alg. 3; solver.py:314-367), device-resident."""
    if ctx.wg is None:
        raise ValidationError("fast scheme needs the mapping compliance built upfront")
    D = frames_tensor(ctx.detection_frames).clone()
    m = D.shape[0]
    c = 3 * m
    p_a = dv.f64(ctx.p_a0).reshape(-1, 3).clone()
    p_b = dv.f64(ctx.p_b0).reshape(-1, 3).clone()
    acc = dv.zeros(c)
    W = dv.square(c)  # 16-byte aligned rows: the pipelined PGS kernel moves W tiles by TMA
    delta = dv.empty(c)
    t = dv.empty(c)
    rot = dv.zeros(1)
    ws = PgsWorkspace(c, pcfg.max_iterations)
    timer = _Timer()
    recs = []
    lam_history = []
    status = _lib.status(acc.device)
    for k in range(ncfg.max_iterations):
        rot_rec = None
        if k > 0 and ncfg.relinearize:
            D, _ = relinearize_device(p_a, p_b, D, rot)
            rot_rec = rot.clone()
            if ncfg.rotation_tol >= 0 and float(rot) <= ncfg.rotation_tol:
                break
        e0 = timer.mark()
        Dm = DirectionMatrix(D)
        rebuild_W_fast(Dm, ctx.wg, out=W)
        e1 = timer.mark()
        compute_violation(Dm, p_a, p_b, out=delta)
        # every iteration keeps its own lambda (lam_history holds references)
        ws_k = ws if k == 0 else PgsWorkspace(c, pcfg.max_iterations)
        res = pgs_device(W, delta, ctx.h, pcfg, ws_k, delta_end=False,
                         colours=ctx.colouring() if pcfg.ordering == "coloured" else None)
        e2 = timer.mark()
        _lib.call("cnb_apply_dt", m, D.data_ptr(), res.lam.data_ptr(), t.data_ptr(), acc.data_ptr(), _lib.stream())
        prox_update_inplace(p_a, p_b, ctx.wg, t, ctx.h)
        # delta_end = delta_base + h^2 W_reg lam (solver.py:201) without a pass over W:
        # the proximity update moved p_a - p_b by h^2 W_g D^T lam, so D (p_a - p_b)
        # is delta_base + h^2 W lam; the regularisation adds h^2 shift_g lam_g
        compute_violation(Dm, p_a, p_b, out=ws_k.delta_end)
        ws_k.delta_end.view(-1, 3).addcmul_(ws_k.shift[:m, None], res.lam.view(-1, 3), value=ctx.h * ctx.h)
        e3 = timer.mark()
        pen = _penetration_device(res.delta_end)
        lam_history.append(res.lam)
        recs.append((e0, e1, e2, e3, res, pen, rot_rec))
        if ncfg.penetration_tol >= 0 and float(pen) <= ncfg.penetration_tol:
            break
    e4 = timer.mark()
    dv_by = mechanical_correction(ctx, acc)
    e5 = timer.mark()
    torch.cuda.current_stream().synchronize()
    status.raise_if_set("newton_fast")
    iters = []
    for e0, e1, e2, e3, res, pen, rot_rec in recs:
        iters.append(IterationStats(
            rebuild_time=timer.secs(e0, e1), pgs_time=timer.secs(e1, e2), correction_time=timer.secs(e2, e3),
            pgs_iterations=res.iterations, pgs_eps=res.eps_history[-1] if res.eps_history else 0.0,
            penetration=float(pen), rotation=float(rot_rec) if rot_rec is not None else 0.0))
    lam_last = lam_history[-1] if lam_history else dv.zeros(c)
    result = CorrectionResult(dv_by, lam_history, LambdaState(lam_last, acc), iters, final_frames=D,
                              final_correction_time=timer.secs(e4, e5))
    result.p_a, result.p_b = p_a, p_b
    return result


def newton_standard(ctx: StepContext, ncfg: NewtonConfig, pcfg: PgsConfig, group=None) -> CorrectionResult:
    """Standard recursive correction (paper Alg. 2; solver.py:260-311).

    Every iteration rebuilds W = sum_o H_o A_o^-1 H_o^T with H_o = D S_o from
    the factorizations (sparse-RHS forward solve + Gram, assemble_W_standard),
    runs PGS, solves dv_k = h A^-1 S^T D^T lam per object and refreshes the
    proximity points through ``ctx.refresh`` (positions g(q_free + h dv)).
    The "single" scheme is this loop with one iteration and no
    re-linearisation (scene.py:701-703).  H_o is formed on the host from the
    iteration's directions (one 9m-double read per iteration).
    """
    from .constraints import assemble_H, assemble_W_standard

    if ctx.refresh is None:
        raise ValidationError("standard scheme needs ctx.refresh (positions from a velocity correction)")
    D = frames_tensor(ctx.detection_frames).clone()
    m = D.shape[0]
    c = 3 * m
    p_a = dv.f64(ctx.p_a0).reshape(-1, 3).clone()
    p_b = dv.f64(ctx.p_b0).reshape(-1, 3).clone()
    dv_tot = {oid: dv.zeros(S.shape[1]) for oid, S in sorted(ctx.S_by_object.items())}
    acc = dv.zeros(c)
    delta = dv.empty(c)
    rot = dv.zeros(1)
    timer = _Timer()
    recs = []
    lam_history = []
    status = _lib.status(acc.device)
    for k in range(ncfg.max_iterations):
        rot_rec = None
        if k > 0 and ncfg.relinearize:
            D, _ = relinearize_device(p_a, p_b, D, rot)
            rot_rec = rot.clone()
            if float(rot) <= ncfg.rotation_tol:
                break
        e0 = timer.mark()
        Dm = DirectionMatrix(D)
        H = {oid: assemble_H(Dm, S) for oid, S in sorted(ctx.S_by_object.items())}
        W = dv.mat64(assemble_W_standard(H, ctx.F_by_object, group=group).W)  # aligned rows for PGS
        e1 = timer.mark()
        compute_violation(Dm, p_a, p_b, out=delta)
        res = pgs_device(W, delta, ctx.h, pcfg, PgsWorkspace(c, pcfg.max_iterations),
                         colours=ctx.colouring() if pcfg.ordering == "coloured" else None)
        e2 = timer.mark()
        t = dv.empty(c)
        _lib.call("cnb_apply_dt", m, D.data_ptr(), res.lam.data_ptr(), t.data_ptr(), acc.data_ptr(), _lib.stream())
        dv_k = mechanical_correction(ctx, t)
        for oid in dv_tot:
            dv_tot[oid] = dv_tot[oid] + dv_k[oid]
        p_a, p_b = ctx.refresh(dv_tot)
        p_a, p_b = p_a.reshape(-1, 3), p_b.reshape(-1, 3)
        e3 = timer.mark()
        pen = _penetration_device(res.delta_end)
        lam_history.append(res.lam)
        recs.append((e0, e1, e2, e3, res, pen, rot_rec))
        if float(pen) <= ncfg.penetration_tol:
            break
    torch.cuda.current_stream().synchronize()
    status.raise_if_set("newton_standard")
    iters = []
    for e0, e1, e2, e3, res, pen, rot_rec in recs:
        iters.append(IterationStats(
            rebuild_time=timer.secs(e0, e1), pgs_time=timer.secs(e1, e2), correction_time=timer.secs(e2, e3),
            pgs_iterations=res.iterations, pgs_eps=res.eps_history[-1] if res.eps_history else 0.0,
            penetration=float(pen), rotation=float(rot_rec) if rot_rec is not None else 0.0))
    lam_last = lam_history[-1] if lam_history else dv.zeros(c)
    result = CorrectionResult(dv_tot, lam_history, LambdaState(lam_last, acc), iters, final_frames=D)
    result.p_a, result.p_b = p_a, p_b
    return result


def newton(ctx: StepContext, ncfg: NewtonConfig, pcfg: PgsConfig) -> CorrectionResult:
    """Dispatch on ``ncfg.scheme`` like Simulation.step (scene.py:696-703)."""
    if ncfg.scheme == "fast":
        return newton_fast(ctx, ncfg, pcfg)
    if ncfg.scheme == "standard":
        return newton_standard(ctx, ncfg, pcfg)
    from dataclasses import replace
    return newton_standard(ctx, replace(ncfg, max_iterations=1, relinearize=False), pcfg)
