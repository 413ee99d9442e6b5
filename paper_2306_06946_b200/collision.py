"""Proximity pairs, contact frames and the geometric mapping.

Mirrors the public surface of the reference module
/root/reference/pkg/src/contactnewton/collision.py.  Frames, re-linearisation,
proximity refresh and signed gaps run on the GPU (contact.cu, pairs.cu);
detection's all-pairs closest-point scan runs on the GPU (detect.cu) with
the reference's selection rule reproduced bit for bit; plane contacts and the
pair records are built on the host.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .errors import DegenerateFrameError, InvalidAttachmentError

COINCIDENT_EPS = 1e-9  # collision.py:24
_TIE_EPS = 1e-9  # collision.py:25


@dataclass
class Pose:
    """x_world = rotation @ x_local + position."""

    rotation: np.ndarray
    position: np.ndarray

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)

    def apply(self, points):
        return np.asarray(points) @ self.rotation.T + self.position

    def inverse_apply(self, points):
        return (np.asarray(points) - self.position) @ self.rotation

    @staticmethod
    def identity() -> "Pose":
        return Pose(np.eye(3), np.zeros(3))


class AttachKind(enum.Enum):
    VERTEX = "vertex"
    BARYCENTRIC = "barycentric"
    RIGID_LOCAL = "rigid_local"
    LOCAL = "local"
    WORLD = "world"


_KIND_CODE = {AttachKind.VERTEX: 0, AttachKind.BARYCENTRIC: 1, AttachKind.RIGID_LOCAL: 2,
              AttachKind.LOCAL: 3, AttachKind.WORLD: 4}
DOF_KINDS = (AttachKind.VERTEX, AttachKind.BARYCENTRIC, AttachKind.RIGID_LOCAL)


@dataclass
class Attachment:
    kind: AttachKind
    object_id: int
    vertex: int = -1
    triangle: np.ndarray | None = None
    weights: np.ndarray | None = None
    local_point: np.ndarray | None = None
    world_point: np.ndarray | None = None
    lever: np.ndarray | None = None
    local_normal: np.ndarray | None = None


@dataclass
class ProximityPair:
    object_a: int
    object_b: int
    attach_a: Attachment
    attach_b: Attachment
    p_a: np.ndarray
    p_b: np.ndarray
    ref_normal: np.ndarray
    signed_distance: float
    vertex_id: int
    element_id: int


@dataclass
class ContactFrame:
    n: np.ndarray
    t1: np.ndarray
    t2: np.ndarray

    def as_matrix(self) -> np.ndarray:
        return np.stack([self.n, self.t1, self.t2])


@dataclass
class MeshGeometry:
    object_id: int
    points: np.ndarray
    triangles: np.ndarray
    vertex_ids: np.ndarray
    deformable: bool
    dynamic: bool
    pose: Pose = field(default_factory=Pose.identity)
    points_dev: torch.Tensor | None = None  # device copy of ``points`` when already resident


@dataclass
class PlaneGeometry:
    object_id: int
    normal: np.ndarray
    offset: float

    def __post_init__(self):
        n = np.asarray(self.normal, dtype=np.float64)
        nn = np.linalg.norm(n)
        if nn == 0:
            raise InvalidAttachmentError("plane normal must be nonzero")
        self.normal = n / nn


# --------------------------------------------------------------------------
# frames as device blocks
# --------------------------------------------------------------------------

class FrameSet:
    """(c_g, 3, 3) device tensor of frames, rows (n, t1, t2); list-like view."""

    def __init__(self, blocks: torch.Tensor):
        self.blocks = blocks

    def __len__(self):
        return self.blocks.shape[0]

    def __getitem__(self, i) -> ContactFrame:
        m = dv.host(self.blocks[i])
        return ContactFrame(m[0].copy(), m[1].copy(), m[2].copy())

    def __iter__(self):
        host = dv.host(self.blocks)
        for m in host:
            yield ContactFrame(m[0].copy(), m[1].copy(), m[2].copy())

    def as_array(self) -> np.ndarray:
        return dv.host(self.blocks)


def frames_tensor(frames) -> torch.Tensor:
    if isinstance(frames, FrameSet):
        return frames.blocks
    if isinstance(frames, torch.Tensor):
        return dv.f64(frames).reshape(-1, 3, 3)
    if len(frames) == 0:
        return dv.zeros((0, 3, 3))
    if isinstance(frames, np.ndarray):
        return dv.f64(frames.reshape(-1, 3, 3))
    return dv.f64(np.stack([f.as_matrix() for f in frames]))


def build_frames(pairs) -> FrameSet:
    """Detection frames (collision.py:359-375) on the device."""
    table = PairTable.of(pairs)
    out = dv.empty((table.m, 3, 3))
    if table.m:
        st = _lib.status(out.device)
        _lib.call("cnb_build_frames", table.m, table.p_a.data_ptr(), table.p_b.data_ptr(),
                  table.ref_normal.data_ptr(), out.data_ptr(), st.ptr, _lib.stream())
        st.raise_if_set("build_frames")
    return FrameSet(out)


def relinearize_device(p_a: torch.Tensor, p_b: torch.Tensor, prev: torch.Tensor,
                       rotation: torch.Tensor | None = None):
    """Re-linearised frames + max rotation, fully on the device (no sync)."""
    m = prev.shape[0]
    out = torch.empty_like(prev)
    rot = rotation if rotation is not None else dv.zeros(1)
    _lib.call("cnb_relinearize", m, p_a.data_ptr(), p_b.data_ptr(), prev.data_ptr(), out.data_ptr(),
              rot.data_ptr(), _lib.stream())
    return out, rot


def relinearize(pairs, p_a, p_b, previous) -> FrameSet:
    """collision.py:381-405 (frames only; rotation via max_frame_rotation)."""
    prev = frames_tensor(previous)
    out, _ = relinearize_device(dv.f64(p_a).reshape(-1, 3), dv.f64(p_b).reshape(-1, 3), prev)
    return FrameSet(out)


def max_frame_rotation(old, new) -> float:
    """collision.py:408-414."""
    a, b = frames_tensor(old), frames_tensor(new)
    if a.shape[0] == 0:
        return 0.0
    c = torch.clamp((a[:, 0, :] * b[:, 0, :]).sum(dim=1), -1.0, 1.0)
    return float(torch.arccos(c).max())


# --------------------------------------------------------------------------
# mapping Jacobian rows (collision.py:417-494)
# --------------------------------------------------------------------------

def _skew(r):
    return np.array([[0.0, -r[2], r[1]], [r[2], 0.0, -r[0]], [-r[1], r[0], 0.0]])


def attachment_triplets(attachment: Attachment, n_dofs: int, row0: int):
    """COO triplets of one attachment's 3 x n_dofs velocity map."""
    rows, cols, vals = [], [], []
    if attachment.kind == AttachKind.VERTEX:
        if not 0 <= 3 * attachment.vertex + 2 < n_dofs:
            raise InvalidAttachmentError(f"vertex {attachment.vertex} out of range")
        for i in range(3):
            rows.append(row0 + i)
            cols.append(3 * attachment.vertex + i)
            vals.append(1.0)
    elif attachment.kind == AttachKind.BARYCENTRIC:
        for node, w in zip(attachment.triangle, attachment.weights):
            if not 0 <= 3 * node + 2 < n_dofs:
                raise InvalidAttachmentError(f"triangle node {node} out of range")
            for i in range(3):
                rows.append(row0 + i)
                cols.append(3 * int(node) + i)
                vals.append(float(w))
    elif attachment.kind == AttachKind.RIGID_LOCAL:
        if n_dofs != 6:
            raise InvalidAttachmentError("rigid attachment on a non-rigid object")
        blk = np.hstack([np.eye(3), -_skew(attachment.lever)])
        for i in range(3):
            for j in range(6):
                if blk[i, j] != 0.0:
                    rows.append(row0 + i)
                    cols.append(j)
                    vals.append(blk[i, j])
    else:
        raise InvalidAttachmentError(f"attachment kind {attachment.kind} carries no DOFs")
    return rows, cols, vals


# --------------------------------------------------------------------------
# device pair table
# --------------------------------------------------------------------------

class PairTable:
    """Structure-of-arrays view of a canonical pair list, on the device.

    Host arrays keep the integer data (for the mapping and bit-exact checks);
    device tensors feed the refresh / gap / frame kernels.
    """

    def __init__(self, pairs: list):
        m = len(pairs)
        self.pairs = pairs
        self.m = m
        kind = np.full((m, 2), 4, dtype=np.int8)
        obj = np.zeros((m, 2), dtype=np.int32)
        node = np.full((m, 2, 3), -1, dtype=np.int64)
        w = np.zeros((m, 2, 3))
        local = np.zeros((m, 2, 3))
        world = np.zeros((m, 2, 3))
        lnormal = np.zeros((m, 3))
        has_ln = np.zeros(m, dtype=np.int8)
        ref = np.zeros((m, 3))
        pa = np.zeros((m, 3))
        pb = np.zeros((m, 3))
        keys = np.zeros((m, 4), dtype=np.int64)
        for i, p in enumerate(pairs):
            for s, at in enumerate((p.attach_a, p.attach_b)):
                kind[i, s] = _KIND_CODE[at.kind]
                obj[i, s] = at.object_id
                if at.kind == AttachKind.VERTEX:
                    node[i, s, 0] = at.vertex
                    w[i, s, 0] = 1.0
                elif at.kind == AttachKind.BARYCENTRIC:
                    node[i, s] = at.triangle
                    w[i, s] = at.weights
                elif at.kind in (AttachKind.LOCAL, AttachKind.RIGID_LOCAL):
                    local[i, s] = at.local_point
                elif at.kind == AttachKind.WORLD:
                    world[i, s] = at.world_point
            if p.attach_b.local_normal is not None:
                lnormal[i] = p.attach_b.local_normal
                has_ln[i] = 1
            ref[i] = p.ref_normal
            pa[i], pb[i] = p.p_a, p.p_b
            keys[i] = (p.object_a, p.object_b, p.vertex_id, p.element_id)
        self.h_kind, self.h_obj, self.h_node, self.h_w = kind, obj, node, w
        self.h_keys = keys
        d = dv.device()
        self.kind = torch.as_tensor(kind, device=d)
        self.obj = torch.as_tensor(obj, device=d)
        self.node = torch.as_tensor(node, device=d)
        self.w = dv.f64(w, d)
        self.local = dv.f64(local, d)
        self.world = dv.f64(world, d)
        self.lnormal = dv.f64(lnormal, d)
        self.has_ln = torch.as_tensor(has_ln, device=d)
        self.ref_normal = dv.f64(ref, d)
        self.p_a = dv.f64(pa, d)
        self.p_b = dv.f64(pb, d)

    @staticmethod
    def of(pairs) -> "PairTable":
        if isinstance(pairs, PairTable):
            return pairs
        return PairTable(list(pairs))

    def participation(self, oid: int):
        """Pairs (ascending) in which object ``oid`` owns a DOF-carrying side, and the side
        (+1 = A, -1 = B)."""
        dof = np.isin(self.h_kind, (0, 1, 2))
        on_a = (self.h_obj[:, 0] == oid) & dof[:, 0]
        on_b = (self.h_obj[:, 1] == oid) & dof[:, 1]
        idx = np.flatnonzero(on_a | on_b)
        side = np.where(on_a[idx], 1, -1).astype(np.int8)
        return idx, side


class PositionViews:
    """Per-object position views for the refresh / gap kernels: a device table of
    node-array pointers (deformable objects) and 3x4 poses (kinematic)."""

    def __init__(self, n_objects: int):
        self.n = n_objects
        self.ptrs = np.zeros(n_objects, dtype=np.int64)
        self.poses = np.zeros((n_objects, 12))
        self.poses[:, [0, 4, 8]] = 1.0
        self._keep = []

    def set_nodes(self, oid: int, q: torch.Tensor):
        self._keep.append(q)
        self.ptrs[oid] = q.data_ptr()

    def set_pose(self, oid: int, pose: Pose):
        self.poses[oid, :9] = pose.rotation.ravel()
        self.poses[oid, 9:] = pose.position

    def device(self):
        d = dv.device()
        return torch.as_tensor(self.ptrs, device=d), dv.f64(self.poses, d)


def refresh_proximity_device(table: PairTable, views: PositionViews, p_a=None, p_b=None):
    """p = g(q) for both sides of every pair (collision.py:497-520), on the device."""
    pa = p_a if p_a is not None else dv.empty((table.m, 3))
    pb = p_b if p_b is not None else dv.empty((table.m, 3))
    if table.m:
        ptrs, poses = views.device()
        _lib.call("cnb_refresh_proximity", table.m, table.kind.data_ptr(), table.obj.data_ptr(),
                  table.node.data_ptr(), table.w.data_ptr(), table.local.data_ptr(),
                  table.world.data_ptr(), ptrs.data_ptr(), poses.data_ptr(), pa.data_ptr(),
                  pb.data_ptr(), _lib.stream())
    return pa, pb


def signed_gaps_device(table: PairTable, views: PositionViews, gaps=None, pen=None):
    """Signed gaps (collision.py:523-548) and pen = max(0, -min gap) (scene.py:658-662)."""
    g = gaps if gaps is not None else dv.empty(table.m)
    p = pen if pen is not None else dv.zeros(1)
    if table.m:
        ptrs, poses = views.device()
        _lib.call("cnb_signed_gaps", table.m, table.kind.data_ptr(), table.obj.data_ptr(),
                  table.node.data_ptr(), table.w.data_ptr(), table.local.data_ptr(),
                  table.world.data_ptr(), table.lnormal.data_ptr(), table.has_ln.data_ptr(),
                  table.ref_normal.data_ptr(), ptrs.data_ptr(), poses.data_ptr(), g.data_ptr(),
                  p.data_ptr(), _lib.stream())
    return g, p


def _views_from_mapping(views: dict) -> PositionViews:
    n = (max(views) + 1) if views else 0
    pv = PositionViews(n)
    for oid, view in views.items():
        if view is None:
            continue
        if isinstance(view, Pose):
            pv.set_pose(oid, view)
        else:
            pv.set_nodes(oid, dv.f64(view).reshape(-1))
    return pv


def refresh_proximity(pairs, views: dict):
    """Reference-shaped wrapper: views = {oid: (n,3) nodes | Pose | None}."""
    table = PairTable.of(pairs)
    return refresh_proximity_device(table, _views_from_mapping(views))


def signed_gaps(pairs, views: dict):
    table = PairTable.of(pairs)
    g, _ = signed_gaps_device(table, _views_from_mapping(views))
    return g


# --------------------------------------------------------------------------
# detection (once per step, before the hot path)
# --------------------------------------------------------------------------

def closest_points_on_triangles(tris: np.ndarray, p: np.ndarray):
    """Ericson closest point of p on every triangle; first true region wins
    (collision.py:138-184)."""
    a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
    ab, ac = b - a, c - a
    ap, bp, cp = p - a, p - b, p - c
    d1 = np.einsum("ij,ij->i", ab, ap)
    d2 = np.einsum("ij,ij->i", ac, ap)
    d3 = np.einsum("ij,ij->i", ab, bp)
    d4 = np.einsum("ij,ij->i", ac, bp)
    d5 = np.einsum("ij,ij->i", ab, cp)
    d6 = np.einsum("ij,ij->i", ac, cp)
    va = d3 * d6 - d5 * d4
    vb = d5 * d2 - d1 * d6
    vc = d1 * d4 - d3 * d2
    with np.errstate(divide="ignore", invalid="ignore"):
        v_ab = np.where(d1 != d3, d1 / (d1 - d3), 0.0)
        w_ac = np.where(d2 != d6, d2 / (d2 - d6), 0.0)
        den_bc = (d4 - d3) + (d5 - d6)
        w_bc = np.where(den_bc != 0, (d4 - d3) / den_bc, 0.0)
        den = va + vb + vc
        v_in = np.where(den != 0, vb / den, 1.0 / 3.0)
        w_in = np.where(den != 0, vc / den, 1.0 / 3.0)
    zero = 0.0 * d1
    conds = [(d1 <= 0) & (d2 <= 0), (d3 >= 0) & (d4 <= d3), (vc <= 0) & (d1 >= 0) & (d3 <= 0),
             (d6 >= 0) & (d5 <= d6), (vb <= 0) & (d2 >= 0) & (d6 <= 0),
             (va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0)]
    v = np.select(conds, [zero, 1.0 + zero, v_ab, zero, zero, 1.0 - w_bc], default=v_in)
    w = np.select(conds, [zero, zero, zero, 1.0 + zero, w_ac, w_bc], default=w_in)
    u = 1.0 - v - w
    return a + v[:, None] * ab + w[:, None] * ac, np.column_stack([u, v, w])


def triangle_normals(tris: np.ndarray) -> np.ndarray:
    n = np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0])
    ln = np.linalg.norm(n, axis=1, keepdims=True)
    return np.divide(n, ln, out=np.zeros_like(n), where=ln > 0)


def _mesh_side(geom: MeshGeometry, vertex=None, triangle=None, bary=None, point=None, normal=None):
    if geom.deformable:
        if vertex is not None:
            return Attachment(AttachKind.VERTEX, geom.object_id, vertex=int(vertex))
        return Attachment(AttachKind.BARYCENTRIC, geom.object_id,
                          triangle=np.asarray(triangle, dtype=np.int64),
                          weights=np.asarray(bary, dtype=np.float64))
    if geom.dynamic:
        raise InvalidAttachmentError("dynamic non-deformable meshes are not supported")
    return Attachment(AttachKind.LOCAL, geom.object_id, local_point=geom.pose.inverse_apply(point),
                      local_normal=None if normal is None else geom.pose.rotation.T @ normal)


def _device_points(geom: MeshGeometry) -> torch.Tensor:
    if geom.points_dev is not None:
        return dv.f64(geom.points_dev).reshape(-1, 3)
    return dv.f64(np.ascontiguousarray(geom.points, dtype=np.float64)).reshape(-1, 3)


def _vertex_vs_mesh(ga: MeshGeometry, gb: MeshGeometry, threshold: float):
    """Best pair per surface vertex of A against B's triangles (collision.py:222-260).

    The all-pairs closest-point scan runs on the GPU (csrc/detect.cu, numpy's
    operation order, bit-exact selection); the host builds the pair records of
    the vertices that pass the threshold gate.
    """
    nv, nt = len(ga.vertex_ids), len(gb.triangles)
    if nv == 0 or nt == 0:
        return []
    d = dv.device()
    vids = torch.as_tensor(np.ascontiguousarray(ga.vertex_ids, dtype=np.int64), device=d)
    tris = torch.as_tensor(np.ascontiguousarray(gb.triangles, dtype=np.int64), device=d)
    pa, pb = _device_points(ga), _device_points(gb)
    work = torch.empty((int(_lib.lib().cnb_detect_work_bytes(nv, nt)) + 7) // 8, dtype=torch.float64, device=d)
    best = torch.empty(nv, dtype=torch.int64, device=d)
    out = torch.empty((nv, 12), dtype=torch.float64, device=d)
    _lib.call("cnb_detect_vertex_mesh", nv, vids.data_ptr(), pa.data_ptr(), nt, tris.data_ptr(), pb.data_ptr(),
              float(threshold), work.data_ptr(), best.data_ptr(), out.data_ptr(), _lib.stream())
    best_h, out_h = best.cpu().numpy(), out.cpu().numpy()
    pts_a = np.asarray(ga.points, dtype=np.float64).reshape(-1, 3)
    res = []
    for q in np.flatnonzero(out_h[:, 11] > 0.0):
        vid, t = int(ga.vertex_ids[q]), int(best_h[q])
        row = out_h[q]
        p, cp, nrm = pts_a[vid], row[5:8].copy(), row[8:11].copy()
        res.append(ProximityPair(
            object_a=ga.object_id, object_b=gb.object_id,
            attach_a=_mesh_side(ga, vertex=vid, point=p),
            attach_b=_mesh_side(gb, triangle=gb.triangles[t], bary=row[2:5].copy(), point=cp, normal=nrm),
            p_a=p.copy(), p_b=cp.copy(), ref_normal=nrm.copy(), signed_distance=float(row[0]), vertex_id=vid,
            element_id=t))
    return res


def _vertex_vs_plane(geom: MeshGeometry, plane: PlaneGeometry, threshold: float):
    n = plane.normal
    pts = geom.points[geom.vertex_ids]
    signed = pts @ n - plane.offset
    out = []
    for k in np.flatnonzero(signed <= threshold):
        vid = int(geom.vertex_ids[k])
        p = geom.points[vid]
        s = float(n @ p - plane.offset)
        foot = p - s * n
        out.append(ProximityPair(
            object_a=geom.object_id, object_b=plane.object_id,
            attach_a=_mesh_side(geom, vertex=vid, point=p),
            attach_b=Attachment(AttachKind.WORLD, plane.object_id, world_point=foot),
            p_a=p.copy(), p_b=foot, ref_normal=n.copy(), signed_distance=s, vertex_id=vid,
            element_id=-1))
    return out


def detect(geometries, threshold: float) -> list:
    """Pairs with signed distance <= threshold in canonical order (collision.py:320-345)."""
    if threshold <= 0:
        raise InvalidAttachmentError(f"threshold must be positive, got {threshold}")
    meshes = [g for g in geometries if isinstance(g, MeshGeometry)]
    planes = [g for g in geometries if isinstance(g, PlaneGeometry)]
    pairs = []
    for ga in meshes:
        for gb in meshes:
            if ga.object_id == gb.object_id or not (ga.dynamic or gb.dynamic):
                continue
            if len(gb.triangles) == 0:
                continue
            lo_a, hi_a = ga.points.min(axis=0), ga.points.max(axis=0)
            lo_b, hi_b = gb.points.min(axis=0), gb.points.max(axis=0)
            if not (np.all(lo_a - threshold <= hi_b) and np.all(lo_b - threshold <= hi_a)):
                continue
            pairs.extend(_vertex_vs_mesh(ga, gb, threshold))
        for plane in planes:
            if ga.dynamic:
                pairs.extend(_vertex_vs_plane(ga, plane, threshold))
    pairs.sort(key=lambda p: (p.object_a, p.object_b, p.vertex_id, p.element_id))
    return pairs
