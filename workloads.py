"""Seeded synthetic inputs of the BASELINE.json configurations.

numpy only: shared by both bench arms, the golden-fixture generator and the
tests.  The reference arm of bench.py builds its scenes from these arrays and
the reference package alone (no import of the B200 package), so the meshes
are generated here rather than by paper_2306_06946_b200.mesh (the two
generators are checked identical in tests/test_workloads_cpu.py).

* five_tet_grid: hexahedral node grid, 5 tets per hex, the two mirror split
  patterns alternating by cell parity so faces conform, every tet positive
  (the reference's box_mesh is the 6-tet Kuhn split).
* cfg1: 40x10x10-node grid (12 000 DoF), 500 barycentric contacts on
  uniformly drawn surface triangles (default_rng(1)), frames from
  default_rng(2), 10 re-draws by 5-degree rotations (default_rng(3)),
  lambda_k ~ U(0, 1) from default_rng(4 + k).
* cfg3: two 50 x 30 x 50-node blocks at 1 cm (450 000 DoF), the upper one
  resting on the lower one.
"""

from __future__ import annotations

import numpy as np

H = 0.01
CFG1_SHAPE = (40, 10, 10)
CFG1_CONTACTS = 500
CFG1_REDRAWS = 10
CFG3_NXZ = 50
CFG3_NY = 30

# corner bit pattern x + 2y + 4z; the odd pattern mirrors the even one
_FIVE_EVEN = np.array([(1, 2, 4, 7), (0, 1, 2, 4), (3, 1, 7, 2), (5, 1, 4, 7), (6, 2, 7, 4)])
_FIVE_ODD = np.array([(0, 3, 5, 6), (1, 0, 5, 3), (2, 0, 3, 6), (4, 0, 6, 5), (7, 3, 6, 5)])
_FACES = np.array([(0, 2, 1), (0, 1, 3), (0, 3, 2), (1, 2, 3)])


def five_tet_grid(shape, spacing=0.01, origin=(0.0, 0.0, 0.0)):
    """(nodes (n, 3), tets (m, 4)) of a shape = (nx, ny, nz)-NODE grid, x fastest."""
    nx, ny, nz = (int(s) for s in shape)
    o = np.asarray(origin, dtype=np.float64)
    s = np.broadcast_to(np.asarray(spacing, dtype=np.float64), (3,))
    gz, gy, gx = np.meshgrid(o[2] + s[2] * np.arange(nz), o[1] + s[1] * np.arange(ny),
                             o[0] + s[0] * np.arange(nx), indexing="ij")
    nodes = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    k, j, i = np.meshgrid(np.arange(nz - 1), np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    bits = np.arange(8)
    corners = (i[:, None] + (bits & 1)) + nx * ((j[:, None] + ((bits >> 1) & 1)) + ny * (k[:, None] + (bits >> 2)))
    odd = ((i + j + k) & 1)[:, None, None] == 1
    tets = np.where(odd, corners[:, _FIVE_ODD], corners[:, _FIVE_EVEN]).reshape(-1, 4)
    a, b, c, d = (nodes[tets[:, q]] for q in range(4))
    flip = np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a) < 0
    tets[flip, 2], tets[flip, 3] = tets[flip, 3].copy(), tets[flip, 2].copy()
    return nodes, tets


def surface_triangles(tets):
    """Outward boundary faces sorted by their oriented node tuple (reference mesh.py:109-122)."""
    faces = np.asarray(tets, dtype=np.int64)[:, _FACES].reshape(-1, 3)
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    once = faces[cnt[inv.ravel()] == 1]
    return once[np.lexsort((once[:, 2], once[:, 1], once[:, 0]))]


def cfg1_inputs():
    nodes, tets = five_tet_grid(CFG1_SHAPE, 0.01)
    tris = surface_triangles(tets)
    rng = np.random.default_rng(1)
    tri_idx = rng.integers(0, len(tris), CFG1_CONTACTS)
    weights = rng.dirichlet((1.0, 1.0, 1.0), CFG1_CONTACTS)
    rng = np.random.default_rng(2)
    frames = np.zeros((CFG1_CONTACTS, 3, 3))
    for i in range(CFG1_CONTACTS):
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        t1 = np.cross(n, rng.standard_normal(3))
        t1 /= np.linalg.norm(t1)
        frames[i] = np.stack([n, t1, np.cross(n, t1)])
    rng = np.random.default_rng(3)
    Ds, cur, ang = [], frames, np.deg2rad(5.0)
    for _ in range(CFG1_REDRAWS):
        ax = rng.standard_normal((CFG1_CONTACTS, 3))
        ax /= np.linalg.norm(ax, axis=1, keepdims=True)
        K = np.zeros((CFG1_CONTACTS, 3, 3))
        K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -ax[:, 2], ax[:, 1], -ax[:, 0]
        K = K - K.transpose(0, 2, 1)
        R = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * (K @ K)
        cur = np.einsum("gij,gkj->gki", R, cur)  # each frame row (direction) rotated
        Ds.append(cur.copy())
    lams = [np.random.default_rng(4 + k).uniform(0.0, 1.0, 3 * CFG1_CONTACTS) for k in range(CFG1_REDRAWS)]
    return dict(nodes=nodes, tets=tets, tris=tris, tri_idx=tri_idx, weights=weights, Ds=Ds, lams=lams)


def cfg3_meshes(nxz=CFG3_NXZ, ny=CFG3_NY, shift=0.0, gap=0.0):
    """Lower and upper block (nodes, tets); the upper block sits ``gap`` above the
    lower's top face, shifted by ``shift`` in x and z."""
    lower = five_tet_grid((nxz, ny, nxz), 0.01)
    top = float(lower[0][:, 1].max())
    upper = five_tet_grid((nxz, ny, nxz), 0.01, (shift, top + gap, shift))
    return lower, upper


# ----------------------------------------------------------------------------
# cfg0 / cfg4: the beam over a tilted plane, and 1 024 seeded copies of it
# ----------------------------------------------------------------------------

CFG0_SHAPE = (20, 4, 4)
CFG4_COPIES = 1024


def plane_normals(tilts_deg):
    """Unit normals (sin t, cos t, 0) of planes tilted by t degrees about z."""
    th = np.deg2rad(np.asarray(tilts_deg, dtype=np.float64))
    return np.stack([np.sin(th), np.cos(th), np.zeros_like(th)], axis=1)


def cfg4_draws(first, count, n_dofs):
    """Copy i: np.random.default_rng([4, i]) -> tilt ~ U(0, 20) deg, mu ~ U(0.2, 0.8),
    then the jitter U(-1e-4, 1e-4) per coordinate."""
    tilts, mus, jit = np.empty(count), np.empty(count), np.empty((count, n_dofs))
    for j in range(count):
        rng = np.random.default_rng([4, first + j])
        tilts[j] = rng.uniform(0.0, 20.0)
        mus[j] = rng.uniform(0.2, 0.8)
        jit[j] = rng.uniform(-1e-4, 1e-4, n_dofs)
    return tilts, mus, jit


def placement(nodes, normals, clearance):
    """(copies, n_nodes, 3): the mesh lifted along y so its lowest node sits
    ``clearance`` above each plane (normal through the origin)."""
    out = np.empty((len(normals),) + nodes.shape)
    for i, nrm in enumerate(normals):
        lift = (clearance - float((nodes @ nrm).min())) / nrm[1]
        out[i] = nodes + np.array([0.0, lift, 0.0])
    return out


# ----------------------------------------------------------------------------
# cfg2: soft ellipsoid pressed by a rotating rigid cylinder
# ----------------------------------------------------------------------------

CFG2_SEMI = (0.10, 0.06, 0.05)
CFG2_SPACING = 0.0035        # jittered lattice spacing: ~30 000 nodes (90 000 DoF)
CFG2_CYL_RADIUS = 0.01
CFG2_INDENT = 0.003          # cylinder's initial indentation into the top (builder's choice)


def ellipsoid_mesh(semi=CFG2_SEMI, spacing=CFG2_SPACING, seed=0):
    """Seeded jittered lattice inside an ellipsoid, Delaunay tets (scipy), tets with
    the centroid outside or a volume below 1e-3 spacing^3 dropped, orientation
    made positive, unused points removed."""
    from scipy.spatial import Delaunay

    rng = np.random.default_rng(seed)
    a = np.asarray(semi, dtype=np.float64)
    axes = [np.arange(-ai, ai + 1e-12, spacing) for ai in a]
    P = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    P = P + rng.uniform(-0.25 * spacing, 0.25 * spacing, P.shape)
    P = P[((P / a) ** 2).sum(axis=1) <= 1.0]
    T = Delaunay(P).simplices.astype(np.int64)
    T = T[((P[T].mean(axis=1) / a) ** 2).sum(axis=1) <= 1.0]
    v = np.einsum("ij,ij->i", np.cross(P[T[:, 1]] - P[T[:, 0]], P[T[:, 2]] - P[T[:, 0]]), P[T[:, 3]] - P[T[:, 0]]) / 6
    T[v < 0] = T[v < 0][:, [0, 2, 1, 3]]
    T = T[np.abs(v) >= 1e-3 * spacing ** 3]
    used = np.unique(T)
    remap = -np.ones(len(P), dtype=np.int64)
    remap[used] = np.arange(len(used))
    return P[used], remap[T]


def cylinder_surface(radius=CFG2_CYL_RADIUS, length=0.12, n_theta=48, n_z=40):
    """Open cylinder side surface along z through the origin, outward wound."""
    th = np.linspace(0.0, 2 * np.pi, n_theta, endpoint=False)
    zs = np.linspace(-0.5 * length, 0.5 * length, n_z + 1)
    pts = np.array([[radius * np.cos(t), radius * np.sin(t), z] for z in zs for t in th])
    tris = []
    for k in range(n_z):
        for j in range(n_theta):
            a, b = k * n_theta + j, k * n_theta + (j + 1) % n_theta
            c, d = a + n_theta, b + n_theta
            tris += [[a, b, d], [a, d, c]]
    tris = np.array(tris, dtype=np.int64)
    n0 = np.cross(pts[tris[:, 1]] - pts[tris[:, 0]], pts[tris[:, 2]] - pts[tris[:, 0]])
    out = pts[tris].mean(axis=1) * np.array([1.0, 1.0, 0.0])
    flip = np.einsum("ij,ij->i", n0, out) < 0
    tris[flip] = tris[flip][:, ::-1]
    return pts, tris


def cfg2_arrays():
    """nodes, tets, fixed (bottom 5 % by y), cylinder points (placed) and triangles,
    cylinder centre."""
    nodes, tets = ellipsoid_mesh()
    fixed = np.sort(np.argsort(nodes[:, 1], kind="stable")[: max(1, len(nodes) // 20)])
    pts, tris = cylinder_surface()
    center = np.array([0.0, float(nodes[:, 1].max()) + CFG2_CYL_RADIUS - CFG2_INDENT, 0.0])
    return nodes, tets, fixed, pts + center, tris, center
