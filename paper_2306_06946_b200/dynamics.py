"""Soft-body mechanics and implicit time integration on the GPU.

Mirrors /root/reference/pkg/src/contactnewton/dynamics.py: ``MechanicalState``
(29-46), ``FreeMotion`` (49-55), ``lame_parameters`` (61-64),
``shape_gradients`` (67-78), ``lumped_masses`` (102-109), ``SoftBody``
(112-211), ``compute_free_motion`` (252-263), ``integrate_correction``
(266-273).

``SoftBody(material="linear")`` is the reference material (K constant, A
factorised once per simulation).  ``material="corotational"`` (north star;
SURVEY.md §9 #1) rotates every element's stiffness by the polar factor of its
deformation gradient, so A changes every step and is refactorised.  Both
assemble with csrc/assembly.cu (one thread per tet, deterministic gathers).
``RigidBody`` (dynamics.py:214-249) is the 6-DoF sphere: its generalized mass
(m I, R I_body R^T) is a 6 x 6 system factorised on the device every step.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _device as dv
from . import _lib
from .errors import NonFiniteForceError, ValidationError
from .linalg import Factorization, SparseSym, SparsityPattern, factorize
from .mesh import TetMesh, check_positive_volumes, tet_volumes

MATERIALS = ("linear", "corotational")


class MechanicalState:
    """Stacked nodal positions q and velocities v (device fp64)."""

    def __init__(self, q, v):
        self.q = dv.f64(q).reshape(-1)
        self.v = dv.f64(v).reshape(-1)
        if self.q.shape != self.v.shape:
            raise ValidationError(f"q and v dimensions disagree: {tuple(self.q.shape)} vs {tuple(self.v.shape)}")

    def copy(self) -> "MechanicalState":
        return MechanicalState(self.q.clone(), self.v.clone())


@dataclass
class FreeMotion:
    dv_free: torch.Tensor
    q_free: torch.Tensor
    factorization: Factorization


def lame_parameters(young: float, poisson: float) -> tuple[float, float]:
    return (young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)),
            young / (2.0 * (1.0 + poisson)))


def shape_gradients(nodes: np.ndarray, tets: np.ndarray):
    """(m, 4, 3) constant shape-function gradients and rest volumes."""
    x0 = nodes[tets[:, 0]]
    E = np.stack([nodes[tets[:, k]] - x0 for k in (1, 2, 3)], axis=2)
    vols = np.linalg.det(E) / 6.0
    inv = np.linalg.inv(E)
    grads = np.empty((len(tets), 4, 3))
    grads[:, 1:, :] = inv
    grads[:, 0, :] = -inv.sum(axis=1)
    return grads, vols


def lumped_masses(nodes: np.ndarray, tets: np.ndarray, density: float) -> np.ndarray:
    masses = np.zeros(len(nodes))
    if len(tets):
        share = density * tet_volumes(nodes, tets) / 4.0
        for k in range(4):
            np.add.at(masses, tets[:, k], share)
    return masses


class _FeLayout:
    """Host-built index maps of one mesh: node-blocked DoF CSR, gather lists."""

    def __init__(self, n_nodes: int, tets: np.ndarray):
        nn = n_nodes
        ne = len(tets)
        # node adjacency incl. self
        if ne:
            a = np.repeat(tets, 4, axis=1).ravel()
            b = np.tile(tets, (1, 4)).ravel()
        else:
            a = b = np.zeros(0, dtype=np.int64)
        a = np.concatenate([a, np.arange(nn)])
        b = np.concatenate([b, np.arange(nn)])
        key = np.unique(a * nn + b)
        bi, bj = key // nn, key % nn  # sorted by (i, j): block ids
        nblk = len(key)
        deg = np.bincount(bi, minlength=nn)
        node_ptr = np.zeros(nn + 1, dtype=np.int64)
        node_ptr[1:] = np.cumsum(deg)
        # DoF CSR: row 3i+d holds 3*deg(i) entries
        row_len = np.repeat(3 * deg, 3)
        rowptr = np.zeros(3 * nn + 1, dtype=np.int64)
        rowptr[1:] = np.cumsum(row_len)
        pos = np.arange(nblk) - node_ptr[bi]  # position of j in i's neighbour list
        cols = (3 * bj[:, None] + np.arange(3)).reshape(-1)  # per block, 3 columns
        # fill column indices row by row
        indices = np.empty(rowptr[-1], dtype=np.int64)
        for d in range(3):
            start = rowptr[3 * bi + d] + 3 * pos
            for e in range(3):
                indices[start + e] = 3 * bj + e
        dst = np.stack([rowptr[3 * bi + d] + 3 * pos for d in range(3)], axis=1)  # (nblk, 3)
        self.rowptr, self.indices = rowptr, indices
        self.dst = dst.reshape(-1)
        self.nblk = nblk
        # element contributions per block, ascending tet
        if ne:
            e_ids = np.repeat(np.arange(ne), 16)
            ab = np.tile(np.arange(16), ne)
            ia = tets[e_ids, ab // 4]
            ib = tets[e_ids, ab % 4]
            blk = np.searchsorted(key, ia * nn + ib)
            order = np.lexsort((e_ids, blk))
            self.contrib = (e_ids * 16 + ab)[order]
            cnt = np.bincount(blk, minlength=nblk)
            # nodes: element forces
            fe_node = tets.reshape(-1)
            forder = np.argsort(fe_node, kind="stable")
            self.fidx = np.arange(ne * 4)[forder]
            fcnt = np.bincount(fe_node, minlength=nn)
        else:
            self.contrib = np.zeros(0, dtype=np.int64)
            cnt = np.zeros(nblk, dtype=np.int64)
            self.fidx = np.zeros(0, dtype=np.int64)
            fcnt = np.zeros(nn, dtype=np.int64)
        self.cptr = np.zeros(nblk + 1, dtype=np.int64)
        self.cptr[1:] = np.cumsum(cnt)
        self.fptr = np.zeros(nn + 1, dtype=np.int64)
        self.fptr[1:] = np.cumsum(fcnt)

    def system_pattern(self, fixed_dof: np.ndarray):
        """Pattern of A given the per-DoF fixed mask (dynamics.py:190-200).

        The reference keeps a K entry only when neither its row nor its
        column is fixed and adds one diagonal entry per DoF; structural zeros
        of the kept 3x3 blocks stay.  Returns (rowptr, indices, src) with
        src[e] = index of A entry e in K's values (-1: a fixed DoF's
        diagonal), or src None when nothing is fixed (A shares K's pattern).
        """
        if not fixed_dof.any():
            return self.rowptr, self.indices, None
        n = len(self.rowptr) - 1
        row = np.repeat(np.arange(n), np.diff(self.rowptr))
        keep = ~(fixed_dof[row] | fixed_dof[self.indices])
        fdof = np.flatnonzero(fixed_dof)
        rows = np.concatenate([row[keep], fdof])
        cols = np.concatenate([self.indices[keep], fdof])
        src = np.concatenate([np.flatnonzero(keep), np.full(len(fdof), -1, dtype=np.int64)])
        order = np.lexsort((cols, rows))
        rowptr = np.zeros(n + 1, dtype=np.int64)
        rowptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
        return rowptr, cols[order].astype(np.int64), src[order].astype(np.int64)


class SoftBody:
    """Tetrahedral FE body (or a tetless particle cloud with explicit masses)."""

    def __init__(self, mesh: TetMesh, young: float = 1e4, poisson: float = 0.3, density: float = 1000.0,
                 rayleigh_mass: float = 0.1, rayleigh_stiffness: float = 0.1, fixed_nodes=None,
                 node_masses=None, extra_node_force=None, material: str = "linear"):
        if young <= 0:
            raise ValidationError(f"young modulus must be positive, got {young}")
        if not 0.0 <= poisson < 0.5:
            raise ValidationError(f"poisson ratio must be in [0, 0.5), got {poisson}")
        if density <= 0:
            raise ValidationError(f"density must be positive, got {density}")
        if material not in MATERIALS:
            raise ValidationError(f"unknown material {material!r}, pick from {MATERIALS}")
        check_positive_volumes(mesh, "soft body")
        self.mesh = mesh
        self.young, self.poisson, self.density = young, poisson, density
        self.rayleigh_mass, self.rayleigh_stiffness = rayleigh_mass, rayleigh_stiffness
        self.material = material
        self.fixed_nodes = np.asarray(fixed_nodes if fixed_nodes is not None else [], dtype=np.int64)
        self.extra_node_force = None if extra_node_force is None else np.asarray(extra_node_force, dtype=np.float64)
        if node_masses is not None:
            node_masses = np.asarray(node_masses, dtype=np.float64)
            if node_masses.shape != (mesh.n_nodes,):
                raise ValidationError("node_masses must list one mass per node")
        elif mesh.n_tets == 0:
            raise ValidationError("a body without tets needs explicit node_masses")
        self.node_masses = node_masses
        self._masses = None
        self._dev = None
        self._gravity_cache = {}

    # -- host properties ------------------------------------------------------------
    @property
    def n_dofs(self) -> int:
        return 3 * self.mesh.n_nodes

    @property
    def fixed_mask(self) -> np.ndarray:
        mask = np.zeros(self.n_dofs, dtype=bool)
        for node in self.fixed_nodes:
            mask[3 * node:3 * node + 3] = True
        return mask

    def masses(self) -> np.ndarray:
        if self._masses is None:
            m = self.node_masses.copy() if self.node_masses is not None else \
                lumped_masses(self.mesh.nodes, self.mesh.tets, self.density)
            if self.mesh.n_nodes and m.min(initial=np.inf) <= 0:
                raise ValidationError("every node needs positive mass")
            self._masses = m
        return self._masses

    # -- device data ------------------------------------------------------------------
    def _device(self):
        if self._dev is None:
            d = dv.device()
            lay = _FeLayout(self.mesh.n_nodes, self.mesh.tets)
            grads, vols = shape_gradients(self.mesh.nodes, self.mesh.tets) if self.mesh.n_tets else \
                (np.zeros((0, 4, 3)), np.zeros(0))
            lam, mu = lame_parameters(self.young, self.poisson)
            ne = self.mesh.n_tets
            D = dict(
                lay=lay, lam=lam, mu=mu, ne=ne,
                rowptr=torch.as_tensor(lay.rowptr, device=d), indices=torch.as_tensor(lay.indices, device=d),
                dst=torch.as_tensor(lay.dst, device=d), cptr=torch.as_tensor(lay.cptr, device=d),
                contrib=torch.as_tensor(lay.contrib, device=d), fptr=torch.as_tensor(lay.fptr, device=d),
                fidx=torch.as_tensor(lay.fidx, device=d),
                tets=torch.as_tensor(self.mesh.tets, device=d), grads=dv.f64(grads, d), vols=dv.f64(vols, d),
                x0=dv.f64(self.mesh.nodes.reshape(-1), d), m3=dv.f64(np.repeat(self.masses(), 3), d),
                fixed=torch.as_tensor(self.fixed_mask.astype(np.int8), device=d),
                Kb=dv.empty((max(ne, 1), 16, 9), d), fe=dv.empty((max(ne, 1), 4, 3), d),
                K=dv.zeros(lay.rowptr[-1], d), Kv=dv.empty(self.n_dofs, d), fel=dv.zeros(self.n_dofs, d),
                R=dv.empty((max(ne, 1), 9), d),
            )
            a_rowptr, a_indices, a_src = lay.system_pattern(self.fixed_mask)
            D["pattern"] = SparsityPattern(a_rowptr, a_indices, self.n_dofs, block_size=3,
                                           coords=self.mesh.nodes)
            if a_src is None:
                D["a_rowptr"], D["a_indices"], D["a_src"] = D["rowptr"], D["indices"], None
            else:
                D["a_rowptr"] = torch.as_tensor(a_rowptr, device=d)
                D["a_indices"] = torch.as_tensor(a_indices, device=d)
                D["a_src"] = torch.as_tensor(a_src, device=d)
            self._dev = D
            if self.material == "linear":
                self._assemble_elements(D["x0"])  # K at rest, constant
        return self._dev

    def _assemble_elements(self, q: torch.Tensor) -> None:
        D = self._dev
        corot = self.material == "corotational"
        st = _lib.stream()
        if D["ne"]:
            _lib.call("cnb_fe_element", D["ne"], D["tets"].data_ptr(), D["grads"].data_ptr(), D["vols"].data_ptr(),
                      q.data_ptr(), D["x0"].data_ptr(), D["lam"], D["mu"], int(corot), D["Kb"].data_ptr(),
                      D["fe"].data_ptr(), D["R"].data_ptr(), st)
        _lib.call("cnb_fe_gather", D["lay"].nblk, D["cptr"].data_ptr(), D["contrib"].data_ptr(), D["Kb"].data_ptr(),
                  D["dst"].data_ptr(), D["K"].data_ptr(), self.mesh.n_nodes, D["fptr"].data_ptr(),
                  D["fidx"].data_ptr(), D["fe"].data_ptr(), D["fel"].data_ptr(), st)

    def _fext(self, gravity) -> torch.Tensor:
        key = tuple(float(x) for x in gravity)
        f = self._gravity_cache.get(key)
        if f is None:
            g = np.asarray(gravity, dtype=np.float64)
            host = np.repeat(self.masses(), 3) * np.tile(g, self.mesh.n_nodes)
            if self.extra_node_force is not None:
                host = host + np.tile(self.extra_node_force, self.mesh.n_nodes)
            f = dv.f64(host)
            self._gravity_cache[key] = f
        return f

    def stiffness(self) -> sp.csr_matrix:
        """Host copy of the current stiffness (rest stiffness for the linear material)."""
        D = self._device()
        return sp.csr_matrix((dv.host(D["K"]), D["lay"].indices, D["lay"].rowptr), shape=(self.n_dofs,) * 2)

    def internal_force(self, q, v) -> torch.Tensor:
        """f(q, v) = f_el(q) + alpha M v + beta K v (dynamics.py:172-177)."""
        D = self._device()
        q, v = dv.f64(q), dv.f64(v)
        self._elastic(q)
        Kv = self._kmul(v, dv.empty(self.n_dofs))
        return D["fel"] + self.rayleigh_mass * (D["m3"] * v) + self.rayleigh_stiffness * Kv

    def _kmul(self, x: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        D = self._dev
        _lib.call("cnb_csr_spmv", self.n_dofs, D["rowptr"].data_ptr(), D["indices"].data_ptr(), D["K"].data_ptr(),
                  x.data_ptr(), out.data_ptr(), 1.0, _lib.stream())
        return out

    def _elastic(self, q: torch.Tensor) -> None:
        """Fill fel (and K for corotational) at configuration q."""
        D = self._dev
        if self.material == "corotational":
            self._assemble_elements(q)
        else:
            disp = q - D["x0"]
            self._kmul(disp, D["fel"])

    def initial_state(self, velocity=(0.0, 0.0, 0.0)) -> MechanicalState:
        v = np.tile(np.asarray(velocity, dtype=np.float64), self.mesh.n_nodes)
        return MechanicalState(self.mesh.nodes.reshape(-1).copy(), v)

    def assemble(self, state: MechanicalState, h: float, gravity, with_matrix: bool = True):
        """(A, b) of backward Euler (dynamics.py:183-211) on the device."""
        if h <= 0:
            raise ValidationError(f"time step must be positive, got {h}")
        D = self._device()
        q, v = dv.f64(state.q), dv.f64(state.v)
        self._elastic(q)
        self._kmul(v, D["Kv"])
        b = dv.empty(self.n_dofs)
        A_vals = dv.empty(D["pattern"].nnz) if with_matrix else None
        st = _lib.status(b.device)
        _lib.call("cnb_fe_system", self.n_dofs, D["a_rowptr"].data_ptr(), D["a_indices"].data_ptr(),
                  D["a_src"].data_ptr() if D["a_src"] is not None else None, D["K"].data_ptr(),
                  D["m3"].data_ptr(), D["fixed"].data_ptr(), float(h), float(self.rayleigh_mass),
                  float(self.rayleigh_stiffness), D["fel"].data_ptr(), D["Kv"].data_ptr(), v.data_ptr(),
                  self._fext(gravity).data_ptr(), A_vals.data_ptr() if A_vals is not None else None, b.data_ptr(),
                  st.ptr, _lib.stream())
        A = SparseSym(pattern=D["pattern"], values=A_vals) if with_matrix else None
        return A, b

    def check_finite(self) -> None:
        try:
            _lib.status(dv.device()).raise_if_set("assemble")
        except _lib.errors.NonFiniteForceError:
            raise NonFiniteForceError("assembled right-hand side is not finite") from None


@dataclass
class RigidBody:
    """Six-DoF rigid body with a sphere as collision geometry (dynamics.py:214-249).
    DoFs: velocity (3) and angular velocity (3) in world axes."""

    mass: float
    inertia: np.ndarray  # (3, 3) body frame, kg m^2
    radius: float = 0.1

    def __post_init__(self):
        if self.mass <= 0:
            raise ValidationError(f"rigid mass must be positive, got {self.mass}")
        self.inertia = np.asarray(self.inertia, dtype=np.float64).reshape(3, 3)
        eig = np.linalg.eigvalsh(0.5 * (self.inertia + self.inertia.T))
        if eig.min() <= 0:
            raise ValidationError("rigid inertia must be symmetric positive definite")

    @property
    def n_dofs(self) -> int:
        return 6

    @property
    def fixed_mask(self) -> np.ndarray:
        return np.zeros(6, dtype=bool)

    def assemble(self, rotation, h: float, gravity):
        """Generalized mass diag(m I, R I R^T) and the gravity impulse (no internal forces)."""
        if h <= 0:
            raise ValidationError(f"time step must be positive, got {h}")
        R = np.asarray(rotation, dtype=np.float64).reshape(3, 3)
        A = np.zeros((6, 6))
        A[:3, :3] = self.mass * np.eye(3)
        A[3:, 3:] = R @ self.inertia @ R.T
        b = np.zeros(6)
        b[:3] = h * self.mass * np.asarray(gravity, dtype=np.float64)
        if not np.all(np.isfinite(b)):
            raise NonFiniteForceError("assembled right-hand side is not finite")
        return SparseSym(sp.csr_matrix(A), check=False), dv.f64(b)

    def check_finite(self) -> None:
        """The right-hand side was checked on the host by ``assemble``."""


def compute_free_motion(A: SparseSym, b, state: MechanicalState, h: float,
                        factorization: Factorization | None = None) -> FreeMotion:
    """dv_free = A^-1 b, q_free = q + h (v + dv_free) (dynamics.py:252-263)."""
    F = factorization if factorization is not None else factorize(A)
    dv_free = F.solve(b)
    q_free = state.q + h * (state.v + dv_free)
    return FreeMotion(dv_free, q_free, F)


def integrate_correction(state: MechanicalState, free: FreeMotion, dv_cor_total, h: float) -> MechanicalState:
    """v+ = v + dv_free + dv_cor, q+ = q_free + h dv_cor (dynamics.py:266-273)."""
    dvc = dv.f64(dv_cor_total)
    return MechanicalState(free.q_free + h * dvc, state.v + free.dv_free + dvc)
