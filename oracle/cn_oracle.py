"""CPU ORACLE — test infrastructure only, never part of the product path.

A numpy/scipy restatement of the reference algorithm for the fast-update
recursive corrective-motion step (paper Alg. 3) of `contactnewton`
(/root/reference/pkg/src/contactnewton).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it, as the checker / CPU baseline.

Every function cites the reference lines it restates.  Data are plain
arrays: a contact set is a dict of structure-of-arrays (``PairSet``) rather
than the reference's dataclass list, but carries the same fields and the same
canonical order.

Third-party arithmetic: the reference factorises with scipy's bundled SuperLU
(`scipy.sparse.linalg.splu`, permc_spec MMD_AT_PLUS_A, diag_pivot_thresh 0,
SymmetricMode; scipy 1.18.1 here, unpinned in the reference's pyproject) —
linalg.py:68-87.  The oracle calls the same routine with the same options.

Pinning: tests/test_oracle_golden.py checks this module against fixtures
generated from the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

# attachment kinds (collision.py:57-62)
VERTEX, BARYCENTRIC, RIGID_LOCAL, LOCAL, WORLD = 0, 1, 2, 3, 4
_DOF_KINDS = (VERTEX, BARYCENTRIC, RIGID_LOCAL)
COINCIDENT_EPS = 1e-9  # collision.py:24
TIE_EPS = 1e-9  # collision.py:25
MAX_TILT_COS = 0.5  # collision.py:378


class OracleError(Exception):
    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# mesh (mesh.py)
# --------------------------------------------------------------------------

_FACES = np.array([(0, 2, 1), (0, 1, 3), (0, 3, 2), (1, 2, 3)])  # mesh.py:106


def tet_volumes(nodes, tets):
    """mesh.py:40-44."""
    a, b, c, d = (nodes[tets[:, k]] for k in range(4))
    return np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a) / 6.0


def surface_triangles(tets):
    """Outward boundary faces sorted by their oriented tuple (mesh.py:109-122)."""
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    if len(tets) == 0:
        return np.zeros((0, 3), dtype=np.int64)
    faces = tets[:, _FACES].reshape(-1, 3)
    keys = np.sort(faces, axis=1)
    _, inv, counts = np.unique(keys, axis=0, return_inverse=True, return_counts=True)
    boundary = faces[counts[inv.ravel()] == 1]
    order = np.lexsort((boundary[:, 2], boundary[:, 1], boundary[:, 0]))
    return boundary[order]


# --------------------------------------------------------------------------
# linear elasticity + backward Euler (dynamics.py)
# --------------------------------------------------------------------------

def lame(young, poisson):
    """dynamics.py:61-64."""
    return (young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)),
            young / (2.0 * (1.0 + poisson)))


def shape_gradients(nodes, tets):
    """dynamics.py:67-78: (m,4,3) gradients and volumes."""
    x0 = nodes[tets[:, 0]]
    E = np.stack([nodes[tets[:, k]] - x0 for k in (1, 2, 3)], axis=2)
    vol = np.linalg.det(E) / 6.0
    Einv = np.linalg.inv(E)
    g = np.empty((len(tets), 4, 3))
    g[:, 1:, :] = Einv
    g[:, 0, :] = -Einv.sum(axis=1)
    return g, vol


def element_blocks(nodes, tets, young, poisson):
    """Per-tet 4x4 blocks of 3x3 (dynamics.py:88-93)."""
    lam, mu = lame(young, poisson)
    g, v = shape_gradients(nodes, tets)
    K = lam * np.einsum("e,eai,ebj->eabij", v, g, g)
    K += mu * np.einsum("e,ebi,eaj->eabij", v, g, g)
    K += mu * np.einsum("e,eab,ij->eabij", v, np.einsum("eai,ebi->eab", g, g), np.eye(3))
    return K


def stiffness(nodes, tets, young, poisson):
    """Global K, COO -> CSR (dynamics.py:81-99)."""
    n = 3 * len(nodes)
    if len(tets) == 0:
        return sp.csr_matrix((n, n))
    K = element_blocks(nodes, tets, young, poisson)
    dof = 3 * tets[:, :, None] + np.arange(3)
    r = np.broadcast_to(dof[:, :, None, :, None], K.shape).ravel()
    c = np.broadcast_to(dof[:, None, :, None, :], K.shape).ravel()
    return sp.coo_matrix((K.ravel(), (r, c)), shape=(n, n)).tocsr()


def lumped_masses(nodes, tets, density):
    """dynamics.py:102-109."""
    m = np.zeros(len(nodes))
    if len(tets):
        share = density * tet_volumes(nodes, tets) / 4.0
        for k in range(4):
            np.add.at(m, tets[:, k], share)
    return m


class Body:
    """Soft body state needed by the oracle (SoftBody dynamics.py:112-211)."""

    def __init__(self, nodes, tets, young=1e4, poisson=0.3, density=1000.0, alpha=0.1, beta=0.1,
                 fixed_nodes=(), node_masses=None, extra_force=None):
        self.x0 = np.asarray(nodes, dtype=np.float64).reshape(-1, 3)
        self.tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
        self.young, self.poisson, self.density = young, poisson, density
        self.alpha, self.beta = alpha, beta
        self.fixed_nodes = np.asarray(fixed_nodes, dtype=np.int64)
        self.masses = (np.asarray(node_masses, dtype=np.float64) if node_masses is not None
                       else lumped_masses(self.x0, self.tets, density))
        self.extra_force = extra_force
        self.K = stiffness(self.x0, self.tets, young, poisson)

    @property
    def n(self):
        return 3 * len(self.x0)

    @property
    def fixed_mask(self):
        mask = np.zeros(self.n, dtype=bool)
        for k in self.fixed_nodes:
            mask[3 * k:3 * k + 3] = True
        return mask

    def internal_force(self, q, v):
        """K(q - q0) + a M v + b K v (dynamics.py:172-177)."""
        m3 = np.repeat(self.masses, 3)
        K = self.stiffness_at(q)
        return self.elastic_force(q) + self.alpha * (m3 * v) + self.beta * (K @ v)

    def stiffness_at(self, q):
        """Stiffness at configuration q (constant for the linear material)."""
        return self.K

    def elastic_force(self, q):
        return self.K @ (q - self.x0.ravel())

    def system(self, q, v, h, gravity):
        """A and b of backward Euler (dynamics.py:183-211)."""
        K = self.stiffness_at(q)
        Kc = K.tocoo()
        m3 = np.repeat(self.masses, 3)
        fx = self.fixed_mask
        keep = ~(fx[Kc.row] | fx[Kc.col])
        diag = np.where(fx, 1.0, (1.0 + h * self.alpha) * m3)
        rows = np.concatenate([Kc.row[keep], np.arange(self.n)])
        cols = np.concatenate([Kc.col[keep], np.arange(self.n)])
        vals = np.concatenate([(h * self.beta + h * h) * Kc.data[keep], diag])
        A = sp.coo_matrix((vals, (rows, cols)), shape=(self.n, self.n)).tocsr()
        f_ext = m3 * np.tile(np.asarray(gravity, dtype=np.float64), len(self.x0))
        if self.extra_force is not None:
            f_ext = f_ext + np.tile(np.asarray(self.extra_force, dtype=np.float64), len(self.x0))
        b = h * (f_ext - self.internal_force(q, v)) - h * h * (K @ v)
        b[fx] = 0.0
        if not np.all(np.isfinite(b)):
            raise OracleError("NonFiniteForce", "rhs not finite")
        return A, b


# --------------------------------------------------------------------------
# corotational material (north star; NOT in the reference)
# --------------------------------------------------------------------------
# The reference material is linear (dynamics.py:165-177): K is assembled once
# and f_el = K (q - q0).  The corotational variant keeps the reference's
# element blocks K_e (dynamics.py:88-93) and its backward-Euler system
# (183-211) but, per tet, rotates them by the rotation R_e of the deformation
# gradient F_e = sum_a x_a g_a^T:
#     K(q)  = sum_e R_e K_e R_e^T,
#     f_el  = sum_e R_e K_e (R_e^T x_e - x0_e),
# and the factorisation is redone every step (the reference caches it for the
# whole simulation, scene.py:411-415).  Parity against the reference itself
# is defined only for the linear material, so this restatement is pinned by
# its own properties (tests/test_oracle_corot_cpu.py): exact reduction to the
# linear material at rest, zero force and rotated K under rigid motions,
# symmetry, and f_el equal to the gradient of the element energy
# 1/2 sum_e u_e^T K_e u_e, u_e = R_e^T x_e - x0_e (finite differences).

def rotation_factor(F):
    """Rotation maximising tr(R^T F) over SO(3) for a stack of 3x3 matrices:
    R = U diag(1, 1, det(U V^T)) V^T.  For det F > 0 this is the orthogonal
    polar factor of F (scipy.linalg.polar's u); for inverted elements the
    reflection is removed along the smallest singular direction."""
    U, _, Vt = np.linalg.svd(F)
    d = np.sign(np.linalg.det(U @ Vt))
    U = U.copy()
    U[..., :, 2] *= d[..., None]
    return U @ Vt


class CorotBody(Body):
    """Corotational soft body: the reference element blocks rotated per tet."""

    refactor_each_step = True

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        self.grads, self.vols = shape_gradients(self.x0, self.tets)
        self.Ke = element_blocks(self.x0, self.tets, self.young, self.poisson)  # (e, a, b, 3, 3)
        dof = 3 * self.tets[:, :, None] + np.arange(3)
        self._r = np.broadcast_to(dof[:, :, None, :, None], self.Ke.shape).ravel()
        self._c = np.broadcast_to(dof[:, None, :, None, :], self.Ke.shape).ravel()

    def rotations(self, q):
        x = np.asarray(q, dtype=np.float64).reshape(-1, 3)
        F = np.einsum("eai,eaj->eij", x[self.tets], self.grads)
        return rotation_factor(F)

    def element_state(self, q):
        """(R (e,3,3), rotated blocks Kb (e,4,4,3,3), element forces fe (e,4,3), local u)."""
        x = np.asarray(q, dtype=np.float64).reshape(-1, 3)
        R = self.rotations(q)
        u = np.einsum("eji,eaj->eai", R, x[self.tets]) - self.x0[self.tets]
        fl = np.einsum("eabij,ebj->eai", self.Ke, u)
        fe = np.einsum("eij,eaj->eai", R, fl)
        Kb = np.einsum("eik,eabkl,ejl->eabij", R, self.Ke, R)
        return R, Kb, fe, u

    def stiffness_at(self, q):
        _, Kb, _, _ = self.element_state(q)
        return sp.coo_matrix((Kb.ravel(), (self._r, self._c)), shape=(self.n, self.n)).tocsr()

    def elastic_force(self, q):
        _, _, fe, _ = self.element_state(q)
        f = np.zeros((len(self.x0), 3))
        np.add.at(f, self.tets.ravel(), fe.reshape(-1, 3))
        return f.ravel()

    def energy(self, q):
        _, _, _, u = self.element_state(q)
        return 0.5 * float(np.einsum("eai,eabij,ebj->", u, self.Ke, u))


class Factor:
    """SuperLU pivot-free symmetric factorisation (linalg.py:68-106)."""

    def __init__(self, A):
        try:
            self.lu = splu(sp.csc_matrix(A), permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                           options=dict(SymmetricMode=True))
        except RuntimeError as exc:
            raise OracleError("NotSPD", str(exc)) from exc
        if not np.all(self.lu.U.diagonal() > 0.0):
            raise OracleError("NotSPD", "non-positive pivot")
        self.dim = A.shape[0]
        self.solves = 0

    def solve(self, b):
        self.solves += 1 if np.ndim(b) == 1 else np.shape(b)[1]
        return self.lu.solve(np.asarray(b, dtype=np.float64))


def naive_gemm(A, B):
    """Ascending-k rank-1 accumulation (linalg.py:121-147)."""
    out = np.zeros((A.shape[0], B.shape[1]))
    for p in range(A.shape[1]):
        out += A[:, p, None] * B[None, p, :]
    return out


# --------------------------------------------------------------------------
# contact sets (collision.py)
# --------------------------------------------------------------------------

def closest_on_triangles(T, p):
    """Ericson closest point, vectorised, first-true region wins (collision.py:138-184)."""
    a, b, c = T[:, 0], T[:, 1], T[:, 2]
    ab, ac = b - a, c - a
    d1 = np.einsum("ij,ij->i", ab, p - a)
    d2 = np.einsum("ij,ij->i", ac, p - a)
    d3 = np.einsum("ij,ij->i", ab, p - b)
    d4 = np.einsum("ij,ij->i", ac, p - b)
    d5 = np.einsum("ij,ij->i", ab, p - c)
    d6 = np.einsum("ij,ij->i", ac, p - c)
    va, vb, vc = d3 * d6 - d5 * d4, d5 * d2 - d1 * d6, d1 * d4 - d3 * d2
    with np.errstate(divide="ignore", invalid="ignore"):
        v_ab = np.where(d1 != d3, d1 / (d1 - d3), 0.0)
        w_ac = np.where(d2 != d6, d2 / (d2 - d6), 0.0)
        dbc = (d4 - d3) + (d5 - d6)
        w_bc = np.where(dbc != 0, (d4 - d3) / dbc, 0.0)
        den = va + vb + vc
        v_in = np.where(den != 0, vb / den, 1.0 / 3.0)
        w_in = np.where(den != 0, vc / den, 1.0 / 3.0)
    z = 0.0 * d1
    regions = [((d1 <= 0) & (d2 <= 0), z, z),
               ((d3 >= 0) & (d4 <= d3), 1.0 + z, z),
               ((vc <= 0) & (d1 >= 0) & (d3 <= 0), v_ab, z),
               ((d6 >= 0) & (d5 <= d6), z, 1.0 + z),
               ((vb <= 0) & (d2 >= 0) & (d6 <= 0), z, w_ac),
               ((va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0), 1.0 - w_bc, w_bc)]
    v = np.select([r[0] for r in regions], [r[1] for r in regions], default=v_in)
    w = np.select([r[0] for r in regions], [r[2] for r in regions], default=w_in)
    u = 1.0 - v - w
    return a + v[:, None] * ab + w[:, None] * ac, np.column_stack([u, v, w])


def unit_normals(T):
    """collision.py:187-190."""
    n = np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0])
    ln = np.linalg.norm(n, axis=1, keepdims=True)
    return np.divide(n, ln, out=np.zeros_like(n), where=ln > 0)


def _empty_pairs():
    return dict(obj_a=[], obj_b=[], kind_a=[], kind_b=[], vert_a=[], tri_b=[], w_b=[],
                local_a=[], local_b=[], world_b=[], lnormal_b=[], p_a=[], p_b=[], ref_normal=[],
                signed=[], vertex_id=[], element_id=[])


def detect(meshes, planes, threshold):
    """Proximity pairs in canonical order (collision.py:221-345).

    meshes: list of dicts(id, points, triangles, vertex_ids, deformable, dynamic,
            pose=(R, t)); planes: list of dicts(id, normal, offset).
    Attachments: side A is a mesh vertex (VERTEX when deformable, else LOCAL),
    side B is BARYCENTRIC / LOCAL on a triangle or WORLD on a plane.
    """
    if threshold <= 0:
        raise OracleError("InvalidAttachment", "threshold must be positive")
    rows = []
    for ga in meshes:
        for gb in meshes:
            if ga["id"] == gb["id"] or not (ga["dynamic"] or gb["dynamic"]):
                continue
            if len(gb["triangles"]) == 0:
                continue
            lo_a, hi_a = ga["points"].min(0), ga["points"].max(0)
            lo_b, hi_b = gb["points"].min(0), gb["points"].max(0)
            if not (np.all(lo_a - threshold <= hi_b) and np.all(lo_b - threshold <= hi_a)):
                continue
            T = gb["points"][gb["triangles"]]
            N = unit_normals(T)
            for vid in ga["vertex_ids"]:
                p = ga["points"][vid]
                cp, bary = closest_on_triangles(T, p)
                diff = p - cp
                dist = np.linalg.norm(diff, axis=1)
                sgn = np.where(np.einsum("ij,ij->i", diff, N) >= 0, dist, -dist)
                best = int(np.flatnonzero(dist <= dist.min() + TIE_EPS).min())
                if sgn[best] > threshold:
                    continue
                rows.append(_mesh_row(ga, gb, int(vid), best, p, cp[best], bary[best], N[best],
                                      float(sgn[best])))
        for pl in planes:
            if not ga["dynamic"]:
                continue
            n = np.asarray(pl["normal"], dtype=np.float64)
            n = n / np.linalg.norm(n)
            for vid in ga["vertex_ids"]:
                p = ga["points"][vid]
                s = float(n @ p - pl["offset"])
                if s > threshold:
                    continue
                rows.append(_plane_row(ga, pl["id"], int(vid), p, n, s))
    rows.sort(key=lambda r: (r["obj_a"], r["obj_b"], r["vertex_id"], r["element_id"]))
    out = _empty_pairs()
    for r in rows:
        for k in out:
            out[k].append(r[k])
    return {k: (np.array(v) if len(v) else np.zeros((0,))) for k, v in out.items()}


def _side_a(ga, vid, p):
    if ga["deformable"]:
        return VERTEX, vid, np.zeros(3)
    R, t = ga["pose"]
    return LOCAL, -1, (p - t) @ R


def _mesh_row(ga, gb, vid, tri, p, cp, bary, normal, signed):
    kind_a, vert_a, local_a = _side_a(ga, vid, p)
    if gb["deformable"]:
        kind_b, local_b, ln = BARYCENTRIC, np.zeros(3), np.full(3, np.nan)
    else:
        if gb["dynamic"]:
            raise OracleError("InvalidAttachment", "dynamic non-deformable mesh")
        R, t = gb["pose"]
        kind_b, local_b, ln = LOCAL, (cp - t) @ R, R.T @ normal
    return dict(obj_a=ga["id"], obj_b=gb["id"], kind_a=kind_a, kind_b=kind_b, vert_a=vert_a,
                tri_b=np.asarray(gb["triangles"][tri], dtype=np.int64), w_b=np.asarray(bary),
                local_a=local_a, local_b=local_b, world_b=np.zeros(3), lnormal_b=ln,
                p_a=p.copy(), p_b=cp.copy(), ref_normal=normal.copy(), signed=signed,
                vertex_id=vid, element_id=tri)


def _plane_row(ga, plane_id, vid, p, n, s):
    kind_a, vert_a, local_a = _side_a(ga, vid, p)
    foot = p - s * n
    return dict(obj_a=ga["id"], obj_b=plane_id, kind_a=kind_a, kind_b=WORLD, vert_a=vert_a,
                tri_b=np.full(3, -1, dtype=np.int64), w_b=np.zeros(3), local_a=local_a,
                local_b=np.zeros(3), world_b=foot, lnormal_b=np.full(3, np.nan), p_a=p.copy(),
                p_b=foot, ref_normal=n.copy(), signed=s, vertex_id=vid, element_id=-1)


def n_pairs(pairs):
    return len(pairs["obj_a"])


def tangents(n):
    """collision.py:351-356."""
    t1 = np.array([1.0, 0.0, 0.0]) - n[0] * n
    if np.linalg.norm(t1) < 1e-6:
        t1 = np.array([0.0, 0.0, 1.0]) - n[2] * n
    t1 = t1 / np.linalg.norm(t1)
    return t1, np.cross(n, t1)


def detection_frames(p_a, p_b, ref_normal):
    """(c,3,3) frames, rows n,t1,t2 (collision.py:359-375)."""
    F = np.zeros((len(p_a), 3, 3))
    for i in range(len(p_a)):
        d = p_a[i] - p_b[i]
        nd = np.linalg.norm(d)
        if nd > COINCIDENT_EPS:
            n = d / nd
            if n @ ref_normal[i] < 0:
                n = -n
        elif np.linalg.norm(ref_normal[i]) > 0.5:
            n = ref_normal[i] / np.linalg.norm(ref_normal[i])
        else:
            raise OracleError("DegenerateFrame", f"pair {i}")
        F[i, 0] = n
        F[i, 1], F[i, 2] = tangents(n)
    return F


def relinearize(p_a, p_b, prev):
    """Frames from the current proximity positions + max rotation (collision.py:381-414)."""
    F = prev.copy()
    worst = 0.0
    for i in range(len(p_a)):
        d = p_a[i] - p_b[i]
        nd = np.linalg.norm(d)
        if nd > COINCIDENT_EPS:
            n = d / nd
            if n @ prev[i, 0] < 0:
                n = -n
            if not n @ prev[i, 0] < MAX_TILT_COS:
                F[i, 0] = n
                F[i, 1], F[i, 2] = tangents(n)
        worst = max(worst, float(np.arccos(np.clip(prev[i, 0] @ F[i, 0], -1.0, 1.0))))
    return F, worst


def mapping_rows(pairs, oid, n_dofs, fixed_mask=None):
    """Signed mapping S_o (constraints.py:101-120 + collision.py:430-462)."""
    m = n_pairs(pairs)
    r, c, v = [], [], []
    for i in range(m):
        for side, sign in (("a", 1.0), ("b", -1.0)):
            if pairs["obj_" + side][i] != oid:
                continue
            kind = pairs["kind_" + side][i]
            if kind == VERTEX:
                node, wts = [pairs["vert_a"][i] if side == "a" else -1], [1.0]
            elif kind == BARYCENTRIC:
                node, wts = list(pairs["tri_b"][i]), list(pairs["w_b"][i])
            else:
                continue
            for nd_, w in zip(node, wts):
                if not 0 <= 3 * nd_ + 2 < n_dofs:
                    raise OracleError("InvalidAttachment", f"node {nd_}")
                for k in range(3):
                    r.append(3 * i + k)
                    c.append(3 * int(nd_) + k)
                    v.append(sign * float(w))
    S = sp.coo_matrix((v, (r, c)), shape=(3 * m, n_dofs)).tocsr()
    if fixed_mask is not None and fixed_mask.any():
        S = S @ sp.diags(np.where(fixed_mask, 0.0, 1.0))
    return S


def attachment_points(pairs, side, q_by_obj, poses):
    """Proximity positions of one side (collision.py:497-520)."""
    m = n_pairs(pairs)
    out = np.empty((m, 3))
    for i in range(m):
        kind, oid = pairs["kind_" + side][i], pairs["obj_" + side][i]
        if kind == VERTEX:
            out[i] = q_by_obj[oid].reshape(-1, 3)[pairs["vert_a"][i]]
        elif kind == BARYCENTRIC:
            out[i] = pairs["w_b"][i] @ q_by_obj[oid].reshape(-1, 3)[pairs["tri_b"][i]]
        elif kind == LOCAL:
            R, t = poses[oid]
            out[i] = pairs["local_" + side][i] @ R.T + t
        else:
            out[i] = pairs["world_b"][i]
    return out


def signed_gaps(pairs, q_by_obj, poses):
    """Gap along the current supporting-element normal (collision.py:523-548)."""
    pa = attachment_points(pairs, "a", q_by_obj, poses)
    pb = attachment_points(pairs, "b", q_by_obj, poses)
    g = np.empty(len(pa))
    for i in range(len(pa)):
        n = pairs["ref_normal"][i]
        if pairs["kind_b"][i] == BARYCENTRIC:
            X = q_by_obj[pairs["obj_b"][i]].reshape(-1, 3)[pairs["tri_b"][i]]
            nn = np.cross(X[1] - X[0], X[2] - X[0])
            if np.linalg.norm(nn) > 0:
                n = nn / np.linalg.norm(nn)
        elif pairs["kind_b"][i] == LOCAL and not np.isnan(pairs["lnormal_b"][i][0]):
            n = poses[pairs["obj_b"][i]][0] @ pairs["lnormal_b"][i]
        g[i] = n @ (pa[i] - pb[i])
    return g


# --------------------------------------------------------------------------
# constraint space (constraints.py) and solver (solver.py)
# --------------------------------------------------------------------------

def block_dense(D):
    c = 3 * len(D)
    out = np.zeros((c, c))
    for g in range(len(D)):
        out[3 * g:3 * g + 3, 3 * g:3 * g + 3] = D[g]
    return out


def mapping_compliance(S_by_obj, F_by_obj):
    """W_g and per-object U_o (constraints.py:155-179)."""
    ids = sorted(S_by_obj)
    dim = S_by_obj[ids[0]].shape[0] if ids else 0
    wg = np.zeros((dim, dim))
    per = {}
    for oid in ids:
        S = S_by_obj[oid]
        if S.nnz == 0:
            per[oid] = np.zeros((dim, dim))
            continue
        U = np.asarray(S @ F_by_obj[oid].solve(S.T.toarray()))
        per[oid] = U
        wg = wg + U
    return wg, per


def rebuild_w(D, wg):
    """D W_g D^T with the naive gemm (constraints.py:182-191)."""
    Dd = block_dense(D)
    return naive_gemm(naive_gemm(Dd, wg), Dd.T)


def violation(D, p_a, p_b):
    """constraints.py:208-214."""
    return np.einsum("gij,gj->gi", D, (p_a - p_b).reshape(-1, 3)).ravel()


def apply_dt(D, lam):
    return np.einsum("gji,gj->gi", D, lam.reshape(-1, 3)).ravel()


def prox_update(p_a, p_b, per_object, D, lam, h, pairs):
    """constraints.py:217-244."""
    t = apply_dt(D, lam)
    p_a, p_b = p_a.copy(), p_b.copy()
    moves = {oid: h * h * (U @ t) for oid, U in per_object.items()}
    for i in range(len(p_a)):
        if pairs["obj_a"][i] in moves:
            p_a[i] += moves[pairs["obj_a"][i]][3 * i:3 * i + 3]
        if pairs["obj_b"][i] in moves:
            p_b[i] -= moves[pairs["obj_b"][i]][3 * i:3 * i + 3]
    return p_a, p_b


def regularize(W):
    """solver.py:99-121."""
    c = W.shape[0]
    if c == 0:
        return W
    shift = 1e-10 * np.trace(W) / c
    if shift <= 0:
        shift = 1e-30
    out = W
    for g in range(c // 3):
        blk = W[3 * g:3 * g + 3, 3 * g:3 * g + 3]
        e = np.linalg.eigvalsh(0.5 * (blk + blk.T))
        if e.min() <= 1e-12 * max(np.abs(e).max(), 1e-300):
            if out is W:
                out = W.copy()
            out[3 * g:3 * g + 3, 3 * g:3 * g + 3] += shift * np.eye(3)
    return out


def local_solve(g, W, dc, lam, mu, h2):
    """solver.py:124-165."""
    i = 3 * g
    if not W[i, i] > 0:
        raise OracleError("SingularBlock", f"group {g}")
    ln_old = lam[i]
    ln = max(0.0, ln_old - dc[i] / (h2 * W[i, i]))
    if ln == 0.0:
        return np.zeros(3)
    if mu == 0.0:
        return np.array([ln, 0.0, 0.0])
    dt = dc[i + 1:i + 3] + h2 * W[i + 1:i + 3, i] * (ln - ln_old)
    T = h2 * W[i + 1:i + 3, i + 1:i + 3]
    det = T[0, 0] * T[1, 1] - T[0, 1] * T[1, 0]
    if not det > 0:
        raise OracleError("SingularBlock", f"group {g} tangential")
    lt = lam[i + 1:i + 3] + np.array([(T[1, 1] * -dt[0] - T[0, 1] * -dt[1]) / det,
                                      (T[0, 0] * -dt[1] - T[1, 0] * -dt[0]) / det])
    nt = float(np.hypot(lt[0], lt[1]))
    if nt > mu * ln:
        lt = lt * (mu * ln / nt)
    return np.array([ln, lt[0], lt[1]])


def pgs(W, delta_base, h, max_iter=30, tol=1e-6, mu=0.5):
    """solver.py:168-202 -> (lam, delta_end, iterations, eps_history, converged)."""
    c = len(delta_base)
    if c == 0:
        return np.zeros(0), np.zeros(0), 0, [], True
    W = regularize(W)
    h2 = h * h
    lam = np.zeros(c)
    dc = np.array(delta_base, dtype=np.float64)
    hist, conv, it = [], False, 0
    for _ in range(max_iter):
        it += 1
        prev = lam.copy()
        for g in range(c // 3):
            new = local_solve(g, W, dc, lam, mu, h2)
            dl = new - lam[3 * g:3 * g + 3]
            if dl.any():
                dc += h2 * (W[:, 3 * g:3 * g + 3] @ dl)
                lam[3 * g:3 * g + 3] = new
        num, den = float(np.linalg.norm(lam - prev)), float(np.linalg.norm(lam))
        eps = 0.0 if num == 0.0 else (np.inf if den == 0.0 else num / den)
        hist.append(eps)
        if eps <= tol:
            conv = True
            break
    return lam, delta_base + h2 * (W @ lam), it, hist, conv


def newton_fast(pairs, frames0, S_by_obj, F_by_obj, p_a0, p_b0, h, wg, per_object, *,
                max_iterations=5, penetration_tol=1e-5, rotation_tol=1e-4, relin=True,
                pgs_iter=30, pgs_tol=1e-6, mu=0.5):
    """solver.py:314-367; returns dict(dv, lam_history, lam, accumulated, frames, rotations,
    pgs_iterations)."""
    D = frames0.copy()
    p_a, p_b = p_a0.copy(), p_b0.copy()
    acc = np.zeros(3 * len(p_a))
    lam_hist, rots, sweeps = [], [], []
    lam_last = np.zeros(3 * len(p_a))
    for k in range(max_iterations):
        rot = 0.0
        if k > 0 and relin:
            D, rot = relinearize(p_a, p_b, D)
            if rot <= rotation_tol:
                break
        W = rebuild_w(D, wg)
        lam, dend, it, _, _ = pgs(W, violation(D, p_a, p_b), h, pgs_iter, pgs_tol, mu)
        p_a, p_b = prox_update(p_a, p_b, per_object, D, lam, h, pairs)
        acc += apply_dt(D, lam)
        lam_hist.append(lam)
        lam_last = lam
        rots.append(rot)
        sweeps.append(it)
        nrm = dend.reshape(-1, 3)[:, 0] if dend.size else np.zeros(0)
        pen = float(max(0.0, -(nrm.min() if nrm.size else 0.0)))
        if pen <= penetration_tol:
            break
    dv = {oid: h * F_by_obj[oid].solve(S_by_obj[oid].T @ acc) for oid in sorted(S_by_obj)}
    return dict(dv=dv, lam_history=lam_hist, lam=lam_last, accumulated=acc, frames=D,
                rotations=rots, pgs_iterations=sweeps, p_a=p_a, p_b=p_b)


# --------------------------------------------------------------------------
# one fast-scheme step for soft bodies over planes (scene.py:608-765)
# --------------------------------------------------------------------------

class Scene:
    """Minimal soft-bodies-on-planes scene advancing with the fast scheme."""

    def __init__(self, bodies, planes, h=0.01, gravity=(0.0, -9.81, 0.0), threshold=0.01,
                 mu=0.5, pgs_iter=30, pgs_tol=1e-6, newton_iter=5, penetration_tol=1e-5,
                 rotation_tol=1e-4, relin=True, velocities=None):
        self.bodies = bodies  # list of Body, object ids 0..len-1; planes follow
        self.planes = planes  # list of dicts(normal, offset); ids assigned after bodies
        self.h, self.g, self.threshold = h, gravity, threshold
        self.cfg = dict(mu=mu, pgs_iter=pgs_iter, pgs_tol=pgs_tol, max_iterations=newton_iter,
                        penetration_tol=penetration_tol, rotation_tol=rotation_tol, relin=relin)
        self.q = [b.x0.ravel().copy() for b in bodies]
        self.v = [np.tile(np.asarray(velocities[i] if velocities else (0, 0, 0), float),
                          len(b.x0)) for i, b in enumerate(bodies)]
        self.tris = [surface_triangles(b.tets) for b in bodies]
        self.factors = [None] * len(bodies)

    def step(self):
        h = self.h
        meshes = []
        for i, b in enumerate(self.bodies):
            tris = self.tris[i]
            vids = np.unique(tris.ravel()) if len(tris) else np.arange(len(b.x0))
            meshes.append(dict(id=i, points=self.q[i].reshape(-1, 3), triangles=tris,
                               vertex_ids=vids, deformable=True, dynamic=True, pose=None))
        planes = [dict(id=len(self.bodies) + k, **p) for k, p in enumerate(self.planes)]
        pairs = detect(meshes, planes, self.threshold)
        m = n_pairs(pairs)
        frames = detection_frames(pairs["p_a"], pairs["p_b"], pairs["ref_normal"]) if m else \
            np.zeros((0, 3, 3))
        F, free_dv, q_free, S = {}, {}, {}, {}
        for i, b in enumerate(self.bodies):
            A, rhs = b.system(self.q[i], self.v[i], h, self.g)
            if self.factors[i] is None or getattr(b, "refactor_each_step", False):
                self.factors[i] = Factor(A)
            F[i] = self.factors[i]
            free_dv[i] = F[i].solve(rhs)
            q_free[i] = self.q[i] + h * (self.v[i] + free_dv[i])
            S[i] = mapping_rows(pairs, i, b.n, b.fixed_mask)
        out = dict(pairs=pairs, frames=frames, n_pairs=m)
        if m:
            p_a0 = attachment_points(pairs, "a", q_free, {})
            p_b0 = attachment_points(pairs, "b", q_free, {})
            out["pen_before"] = float(max(0.0, -signed_gaps(pairs, q_free, {}).min()))
            wg, per = mapping_compliance(S, F)
            res = newton_fast(pairs, frames, S, F, p_a0, p_b0, h, wg, per, **self.cfg)
            dv = res["dv"]
            out.update(wg=wg, p_a0=p_a0, p_b0=p_b0, result=res)
        else:
            dv = {i: np.zeros(b.n) for i, b in enumerate(self.bodies)}
            out["pen_before"] = 0.0
        for i in range(len(self.bodies)):
            self.v[i] = self.v[i] + free_dv[i] + dv[i]
            self.q[i] = q_free[i] + h * dv[i]
        out["pen_after"] = float(max(0.0, -signed_gaps(pairs, dict(enumerate(self.q)), {}).min())) \
            if m else 0.0
        return out
