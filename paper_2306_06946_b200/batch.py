"""Batched independent scenes: BASELINE configs[4].

Many copies of one soft body (shared mesh and linear material, so one system
matrix A and one factorisation) each falling onto its own plane with its own
friction coefficient and initial jitter.  Every copy follows the reference's
``Simulation.step`` with the fast scheme (scene.py:608-765): vertex-plane
detection (collision.py:264-287), free motion (dynamics.py:252-263), W_g
(constraints.py:155-179), ``max_iterations`` forced corrective iterations of
[re-linearise, W = D W_g D^T, violation, PGS, proximity update]
(solver.py:314-367), mechanical correction and integration
(solver.py:250-257, dynamics.py:266-273).

B200 mapping: all copies advance together.  A is shared and constant, so its
inverse is formed once from the GPU Cholesky factor; the per-step multi-RHS
solves of all copies are one fp64 tensor-core GEMM each, and W_g of every copy
is a gather from the inverse (a vertex-plane row of S is a unit row).  The
per-pair kernels run on the concatenated pairs of all copies, rebuild / PGS /
proximity update run per copy in one launch (csrc/batch.cu, pgs_batched_kernel:
one CTA per copy).  Multi-GPU: copies are split across ranks, no collective on
the data path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .dynamics import SoftBody
from .linalg import Factorization
from .mesh import surface_triangles


def plane_normals(tilts_deg) -> np.ndarray:
    """Unit normals (sin t, cos t, 0) of planes tilted by t degrees about z."""
    th = np.deg2rad(np.asarray(tilts_deg, dtype=np.float64))
    return np.stack([np.sin(th), np.cos(th), np.zeros_like(th)], axis=1)


def cfg4_draws(first: int, count: int, n_dofs: int):
    """Per-copy draws of BASELINE configs[4]: copy i uses
    ``np.random.default_rng([4, i])`` for tilt ~ U(0, 20) degrees, then
    mu ~ U(0.2, 0.8), then the jitter U(-1e-4, 1e-4) per coordinate."""
    tilts, mus, jit = np.empty(count), np.empty(count), np.empty((count, n_dofs))
    for j in range(count):
        rng = np.random.default_rng([4, first + j])
        tilts[j] = rng.uniform(0.0, 20.0)
        mus[j] = rng.uniform(0.2, 0.8)
        jit[j] = rng.uniform(-1e-4, 1e-4, n_dofs)
    return tilts, mus, jit


def placement(nodes: np.ndarray, normals: np.ndarray, clearance: float) -> np.ndarray:
    """(ns, n_nodes, 3): the mesh translated along y so that its lowest node sits
    ``clearance`` above each plane (normal through the origin)."""
    out = np.empty((len(normals),) + nodes.shape)
    for i, nrm in enumerate(normals):
        lift = (clearance - float((nodes @ nrm).min())) / nrm[1]
        out[i] = nodes + np.array([0.0, lift, 0.0])
    return out


class BatchedPlaneScenes:
    """``ns`` copies of ``mesh`` over tilted planes (normal (sin t, cos t, 0) through
    the origin); the lowest node of copy i starts ``clearance`` above its plane.

    tilts_deg, mus: per-copy plane tilt (degrees) and friction; jitter: (ns, 3 n_nodes)
    added to the initial positions (applied to the state, not the rest shape, as the
    reference's tests do); rest_nodes: (ns, n_nodes, 3) explicit per-copy rest shapes
    (translates of ``mesh``) instead of the placement; normals: (ns, 3) explicit plane
    normals instead of the tilts."""

    def __init__(self, mesh, tilts_deg, mus, jitter=None, *, young=5e3, poisson=0.45, density=1000.0,
                 rayleigh_mass=0.1, rayleigh_stiffness=0.1, h=0.01, gravity=(0.0, -9.81, 0.0), threshold=0.005,
                 newton_iterations=5, pgs_tolerance=1e-10, pgs_max_iterations=1000, clearance=0.02,
                 rest_nodes=None, normals=None):
        self.ns = ns = len(tilts_deg)
        self.h, self.gravity, self.threshold = float(h), tuple(gravity), float(threshold)
        self.newton_iterations = int(newton_iterations)
        self.pgs_tol, self.pgs_max = float(pgs_tolerance), int(pgs_max_iterations)
        self.body = SoftBody(mesh, young=young, poisson=poisson, density=density, rayleigh_mass=rayleigh_mass,
                             rayleigh_stiffness=rayleigh_stiffness, material="linear")
        if self.body.fixed_mask.any():
            raise ValueError("batched scenes: fixed nodes are not supported (unit-row mapping)")
        n = self.n = self.body.n_dofs
        normals = plane_normals(tilts_deg) if normals is None else np.asarray(normals, dtype=np.float64)
        self.mus = np.asarray(mus, dtype=np.float64)
        if rest_nodes is None:
            rest_nodes = placement(mesh.nodes, normals, clearance)
        self.rest_host = np.ascontiguousarray(rest_nodes, dtype=np.float64).reshape(ns, n)
        q0 = self.rest_host.copy()
        if jitter is not None:
            q0 = q0 + np.asarray(jitter, dtype=np.float64).reshape(ns, n)
        self.q0_host = q0
        d = dv.device()
        self.X0 = dv.f64(self.rest_host)  # per-copy rest shape (translated mesh)
        self.Q = dv.f64(q0)
        self.V = dv.zeros((ns, n))
        self.normals = dv.f64(normals)
        self.offsets = dv.zeros(ns)
        self.vids_host = np.unique(surface_triangles(mesh)).astype(np.int64)
        self.vids = torch.as_tensor(self.vids_host, device=d)
        self.nsurf = len(self.vids_host)
        # shared system matrix, factor and inverse
        st0 = self.body.initial_state()
        A, _ = self.body.assemble(st0, self.h, self.gravity)
        self.F = Factorization(A)
        eye = torch.eye(n, dtype=torch.float64, device=d)
        Ainv = self.F.solve_device(eye)  # rows = A^-1 e_j
        self.Ainv = (0.5 * (Ainv + Ainv.t())).contiguous()  # exactly symmetric, W_g blocks symmetric
        del Ainv, eye
        D = self.body._device()
        self._rowptr, self._indices, self._K = D["rowptr"], D["indices"], D["K"]
        self._m3, self._fixed = D["m3"], D["fixed"]
        self._fext = self.body._fext(self.gravity)
        self.time = 0.0
        self.step_index = 0
        self._prev_sweeps = None
        self._bufs = {}
        self._status = _lib.status(d)
        self.last = {}

    # -- helpers -------------------------------------------------------------------
    def _resident(self, name: str, size: int) -> torch.Tensor:
        """A view of a grow-only resident buffer (the per-copy W_g / W blocks: the
        contact count drifts by a few pairs between steps; reallocating hundreds of
        MB then would stall the step)."""
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < size:
            buf = dv.empty(max(int(size * 1.25), 1))
            self._bufs[name] = buf
        return buf[:size]

    def _solve(self, B: torch.Tensor) -> torch.Tensor:
        """X (ns, n) with A x_s = b_s for every copy: one DMMA GEMM with the inverse."""
        X = torch.empty_like(B)
        _lib.call("cnb_gemm_dense", B.shape[0], self.n, self.n, B.data_ptr(), self.n, self.Ainv.data_ptr(), self.n,
                  X.data_ptr(), self.n, _lib.stream())
        return X

    def _rhs(self) -> torch.Tensor:
        ns, n = self.ns, self.n
        disp = self.Q - self.X0
        fel, Kv, b = dv.empty((ns, n)), dv.empty((ns, n)), dv.empty((ns, n))
        st = _lib.stream()
        for x, y in ((disp, fel), (self.V, Kv)):
            _lib.call("cnb_batch_spmv", ns, n, self._rowptr.data_ptr(), self._indices.data_ptr(), self._K.data_ptr(),
                      x.data_ptr(), n, y.data_ptr(), n, st)
        _lib.call("cnb_batch_rhs", ns, n, fel.data_ptr(), Kv.data_ptr(), self._m3.data_ptr(), self.V.data_ptr(),
                  self._fext.data_ptr(), self._fixed.data_ptr(), self.h, float(self.body.rayleigh_mass),
                  float(self.body.rayleigh_stiffness), b.data_ptr(), self._status.ptr, st)
        return b

    def _detect(self):
        """Pairs of every copy in canonical order; host gets only the per-copy counts."""
        ns, d = self.ns, dv.device()
        st = _lib.stream()
        count = torch.empty(ns, dtype=torch.int32, device=d)
        kept = torch.empty((ns, self.nsurf), dtype=torch.int32, device=d)
        _lib.call("cnb_batch_detect_planes", ns, self.nsurf, self.vids.data_ptr(), self.Q.data_ptr(), self.n,
                  self.normals.data_ptr(), self.offsets.data_ptr(), self.threshold, count.data_ptr(), kept.data_ptr(),
                  st)
        cnt = count.cpu().numpy().astype(np.int64)
        poff = np.zeros(ns + 1, dtype=np.int64)
        poff[1:] = np.cumsum(cnt)
        m = int(poff[-1])
        boff = np.zeros(ns + 1, dtype=np.int64)
        boff[1:] = np.cumsum(cnt * cnt)
        ldw = 3 * cnt + (cnt & 1)  # even row stride: 16-byte aligned rows of W_g / W
        woff = np.zeros(ns + 1, dtype=np.int64)
        woff[1:] = np.cumsum(ldw * ldw)
        P = dict(m=m, poff_h=poff, boff_h=boff, woff_h=woff, cnt=cnt, wsize=int(woff[-1]),
                 poff=dv.upload(poff), boff=dv.upload(boff), woff=dv.upload(woff))
        P["scene"] = torch.empty(m, dtype=torch.int32, device=d)
        P["cand"] = torch.empty(m, dtype=torch.int32, device=d)
        P["pa"], P["pb"], P["ref"] = dv.empty((m, 3)), dv.empty((m, 3)), dv.empty((m, 3))
        P["signed"] = dv.empty(m)
        _lib.call("cnb_batch_pairs", ns, m, self.nsurf, P["poff"].data_ptr(), kept.data_ptr(), self.vids.data_ptr(),
                  self.Q.data_ptr(), self.n, self.normals.data_ptr(), self.offsets.data_ptr(), P["scene"].data_ptr(),
                  P["cand"].data_ptr(), P["pa"].data_ptr(), P["pb"].data_ptr(), P["ref"].data_ptr(),
                  P["signed"].data_ptr(), st)
        return P

    # -- one time step of every copy ----------------------------------------------------
    def step(self):
        ns, n, h = self.ns, self.n, self.h
        st = _lib.stream()
        if self.last.get("iters_all"):
            # after the previous step (its kernels are done once detection syncs below)
            self._pending_sweeps = self.last["iters_all"][0]
        P = self._detect()
        if getattr(self, "_pending_sweeps", None) is not None:
            self._prev_sweeps = self._pending_sweeps[:, 0].cpu().numpy().astype(np.float64)
            self._pending_sweeps = None
        m = P["m"]
        # free motion
        dv_free = self._solve(self._rhs())
        q_free = self.Q + h * (self.V + dv_free)
        acc = dv.zeros(3 * m)
        if m:
            # frames from detection, proximity points from the free motion
            D = dv.empty((m, 3, 3))
            _lib.call("cnb_build_frames", m, P["pa"].data_ptr(), P["pb"].data_ptr(), P["ref"].data_ptr(),
                      D.data_ptr(), self._status.ptr, st)
            pa = dv.empty((m, 3))
            _lib.call("cnb_batch_gather_pa", m, P["scene"].data_ptr(), P["cand"].data_ptr(), self.vids.data_ptr(),
                      q_free.data_ptr(), n, pa.data_ptr(), st)
            pb = P["pb"]  # world points on the planes
            nblk = int(P["boff_h"][-1])
            Wg, W = self._resident("Wg", P["wsize"]), self._resident("W", P["wsize"])
            _lib.call("cnb_batch_wg_gather", ns, nblk, P["boff"].data_ptr(), P["poff"].data_ptr(),
                      P["woff"].data_ptr(), P["cand"].data_ptr(), self.vids.data_ptr(), self.Ainv.data_ptr(), n,
                      Wg.data_ptr(), st)
            delta, t = dv.empty(3 * m), dv.empty(3 * m)
            lam = dv.empty(3 * m)  # (delta_end is not needed: the proximity update follows)
            eps = dv.empty((ns, self.pgs_max))
            ics = []
            rot = dv.zeros(1)
            g_off = np.ascontiguousarray(P["poff_h"])
            order = self._launch_order(P["cnt"])
            w_off = np.ascontiguousarray(P["woff_h"][:-1])
            mus = np.ascontiguousarray(self.mus)
            Dk = D
            for k in range(self.newton_iterations):
                if k > 0:  # re-linearise from the current proximity points (collision.py:381-405)
                    Dn = dv.empty((m, 3, 3))
                    _lib.call("cnb_relinearize", m, pa.data_ptr(), pb.data_ptr(), Dk.data_ptr(), Dn.data_ptr(),
                              rot.data_ptr(), st)
                    Dk = Dn
                _lib.call("cnb_batch_rebuild_w", ns, nblk, P["boff"].data_ptr(), P["poff"].data_ptr(),
                          P["woff"].data_ptr(), Dk.data_ptr(), Wg.data_ptr(), W.data_ptr(), st)
                _lib.call("cnb_violation", m, Dk.data_ptr(), pa.data_ptr(), pb.data_ptr(), delta.data_ptr(), st)
                ic = torch.zeros((ns, 2), dtype=torch.int32, device=dv.device())
                ics.append(ic)
                _lib.call("cnb_pgs_batched", ns, g_off.ctypes.data, w_off.ctypes.data, mus.ctypes.data, W.data_ptr(),
                          delta.data_ptr(), h, self.pgs_tol, self.pgs_max, lam.data_ptr(), None,
                          eps.data_ptr(), ic.data_ptr(), order.ctypes.data, self._status.ptr, st)
                _lib.call("cnb_apply_dt", m, Dk.data_ptr(), lam.data_ptr(), t.data_ptr(), acc.data_ptr(), st)
                _lib.call("cnb_batch_prox", ns, m, P["poff"].data_ptr(), P["woff"].data_ptr(), Wg.data_ptr(),
                          t.data_ptr(), h, pa.data_ptr(), st)
            self.last = dict(pairs=P, lam=lam, frames=Dk, iters=ic, iters_all=ics, pa=pa)
        # mechanical correction dv = h A^-1 S^T acc, integration
        rhs = dv.zeros((ns, n))
        if m:
            _lib.call("cnb_batch_scatter_acc", m, P["scene"].data_ptr(), P["cand"].data_ptr(), self.vids.data_ptr(),
                      acc.data_ptr(), rhs.data_ptr(), n, st)
        dv_cor = self._solve(rhs).mul_(h)
        self.Q = q_free + h * dv_cor
        self.V = self.V + dv_free + dv_cor
        self.time += h
        self.step_index += 1
        return m

    def _launch_order(self, cnt):
        """Batched-PGS launch order: expected work (the previous step's first-iteration
        sweeps, which dominate, times c_s^2) descending, so the longest solves start
        first; the previous step's counts are complete once this step's detection has
        synchronised."""
        prev = self._prev_sweeps
        if os.environ.get("CNB_BATCH_ORDER", "1") == "0":  # diagnostic: launch in copy order
            return np.arange(len(cnt), dtype=np.int32)
        work = cnt.astype(np.float64) ** 2 * (prev if prev is not None else 1.0)
        return np.ascontiguousarray(np.argsort(-work, kind="stable").astype(np.int32))

    def check(self):
        """Raise the reference's exception for a device-side failure (synchronises)."""
        torch.cuda.current_stream().synchronize()
        self._status.raise_if_set("batched scenes")

    def pair_keys(self, scene: int) -> np.ndarray:
        """Vertex ids of the last step's pairs of one copy (canonical order)."""
        P = self.last["pairs"]
        a, b = int(P["poff_h"][scene]), int(P["poff_h"][scene + 1])
        return self.vids_host[P["cand"][a:b].cpu().numpy()]
