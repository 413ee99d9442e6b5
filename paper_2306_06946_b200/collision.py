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


@dataclass
class SphereGeometry:
    """A rigid sphere for detection (collision.py:127-132): centre, radius and the
    body pose its contact points are expressed in."""

    object_id: int
    center: np.ndarray
    radius: float
    pose: Pose
    dynamic: bool = True


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
    """COO triplets (rows, cols, vals) of one attachment's 3 x n_dofs velocity map
    (reference collision.py:430-462).

    A point attached to nodes k with weights w moves with sum_k w_k v_k, so node
    k contributes w_k I_3 at columns 3k..3k+2 (VERTEX: one node, weight 1;
    BARYCENTRIC: the triangle's nodes).  A rigid lever r maps the 6 body DoFs
    through [I_3, -skew(r)] (its nonzeros, row-major).  Entries come out row
    block by row block in node order, the reference's triplet order.
    """
    kind = attachment.kind
    if kind == AttachKind.RIGID_LOCAL:
        if n_dofs != 6:
            raise InvalidAttachmentError("rigid attachment on a non-rigid object")
        jac = np.concatenate([np.eye(3), -_skew(attachment.lever)], axis=1)
        r, c = np.nonzero(jac)
        return (row0 + r).tolist(), c.tolist(), jac[r, c].tolist()
    if kind == AttachKind.VERTEX:
        nodes, weights, what = np.array([int(attachment.vertex)]), np.ones(1), "vertex"
    elif kind == AttachKind.BARYCENTRIC:
        nodes = np.asarray(attachment.triangle, dtype=np.int64).reshape(-1)
        weights, what = np.asarray(attachment.weights, dtype=np.float64).reshape(-1), "triangle node"
    else:
        raise InvalidAttachmentError(f"attachment kind {attachment.kind} carries no DOFs")
    bad = (nodes < 0) | (3 * nodes + 2 >= n_dofs)
    if bad.any():
        raise InvalidAttachmentError(f"{what} {int(nodes[bad][0])} out of range")
    rows = row0 + np.tile(np.arange(3), len(nodes))
    cols = (3 * nodes[:, None] + np.arange(3)).reshape(-1)
    return rows.tolist(), cols.tolist(), np.repeat(weights, 3).tolist()


# --------------------------------------------------------------------------
# device pair table
# --------------------------------------------------------------------------

class PairSoA:
    """Structure-of-arrays pair records as detection produces them (canonical order
    after ``sort``); ``LazyPairs`` turns rows into ``ProximityPair`` objects on demand,
    ``PairTable.from_soa`` uploads them without building Python objects."""

    FIELDS = ("kind", "obj", "node", "w", "local", "world", "lnormal", "has_ln", "ref", "pa", "pb", "signed",
              "keys", "lever")

    def __init__(self, m: int = 0):
        self.kind = np.full((m, 2), 4, dtype=np.int8)
        self.obj = np.zeros((m, 2), dtype=np.int32)
        self.node = np.full((m, 2, 3), -1, dtype=np.int64)
        self.w = np.zeros((m, 2, 3))
        self.local = np.zeros((m, 2, 3))
        self.world = np.zeros((m, 2, 3))
        self.lnormal = np.zeros((m, 3))
        self.has_ln = np.zeros(m, dtype=np.int8)
        self.ref = np.zeros((m, 3))
        self.pa = np.zeros((m, 3))
        self.pb = np.zeros((m, 3))
        self.signed = np.zeros(m)
        self.keys = np.zeros((m, 4), dtype=np.int64)
        self.lever = np.zeros((m, 3))  # RIGID_LOCAL side A: contact point minus the body centre

    def __len__(self) -> int:
        return len(self.keys)

    @staticmethod
    def concat(parts) -> "PairSoA":
        out = PairSoA(0)
        parts = [q for q in parts if len(q)]
        if parts:
            for f in PairSoA.FIELDS:
                setattr(out, f, np.concatenate([getattr(q, f) for q in parts]))
        return out

    def take(self, order) -> "PairSoA":
        out = PairSoA(0)
        for f in PairSoA.FIELDS:
            setattr(out, f, getattr(self, f)[order])
        return out

    def sort(self) -> "PairSoA":
        """Canonical order (collision.py:344): (object_a, object_b, vertex_id, element_id)."""
        k = self.keys
        return self.take(np.lexsort((k[:, 3], k[:, 2], k[:, 1], k[:, 0])))

    def attachment(self, i: int, s: int) -> Attachment:
        kind = int(self.kind[i, s])
        oid = int(self.obj[i, s])
        if kind == 0:
            return Attachment(AttachKind.VERTEX, oid, vertex=int(self.node[i, s, 0]))
        if kind == 1:
            return Attachment(AttachKind.BARYCENTRIC, oid, triangle=self.node[i, s].copy(), weights=self.w[i, s].copy())
        if kind == 2:
            return Attachment(AttachKind.RIGID_LOCAL, oid, local_point=self.local[i, s].copy(),
                              lever=self.lever[i].copy())
        if kind == 3:
            ln = self.lnormal[i].copy() if (s == 1 and self.has_ln[i]) else None
            return Attachment(AttachKind.LOCAL, oid, local_point=self.local[i, s].copy(), local_normal=ln)
        return Attachment(AttachKind.WORLD, oid, world_point=self.world[i, s].copy())

    def pair(self, i: int) -> ProximityPair:
        k = self.keys[i]
        return ProximityPair(object_a=int(k[0]), object_b=int(k[1]), attach_a=self.attachment(i, 0),
                             attach_b=self.attachment(i, 1), p_a=self.pa[i].copy(), p_b=self.pb[i].copy(),
                             ref_normal=self.ref[i].copy(), signed_distance=float(self.signed[i]),
                             vertex_id=int(k[2]), element_id=int(k[3]))


class LazyPairs:
    """Read-only sequence of ``ProximityPair`` backed by a ``PairSoA`` (objects are
    built on first access: a step never needs them)."""

    def __init__(self, soa: PairSoA):
        self.soa = soa
        self._cache = {}

    def __len__(self) -> int:
        return len(self.soa)

    def __bool__(self) -> bool:
        return len(self.soa) > 0

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        p = self._cache.get(i)
        if p is None:
            p = self._cache[i] = self.soa.pair(i)
        return p

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


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
        self.kind = dv.upload(kind)
        self.obj = dv.upload(obj)
        self.node = dv.upload(node)
        self.w = dv.f64(w, d)
        self.local = dv.f64(local, d)
        self.world = dv.f64(world, d)
        self.lnormal = dv.f64(lnormal, d)
        self.has_ln = dv.upload(has_ln)
        self.ref_normal = dv.f64(ref, d)
        self.p_a = dv.f64(pa, d)
        self.p_b = dv.f64(pb, d)

    @classmethod
    def from_soa(cls, soa: PairSoA) -> "PairTable":
        """Table straight from detection arrays (no per-pair Python objects)."""
        self = cls.__new__(cls)
        self.soa = soa
        self.pairs = LazyPairs(soa)
        self.m = len(soa)
        self.h_kind, self.h_obj, self.h_node, self.h_w = soa.kind, soa.obj, soa.node, soa.w
        self.h_keys = soa.keys
        d = dv.device()
        self.kind = dv.upload(soa.kind)
        self.obj = dv.upload(soa.obj)
        self.node = dv.upload(soa.node)
        self.w = dv.f64(soa.w, d)
        self.local = dv.f64(soa.local, d)
        self.world = dv.f64(soa.world, d)
        self.lnormal = dv.f64(soa.lnormal, d)
        self.has_ln = dv.upload(soa.has_ln)
        self.ref_normal = dv.f64(soa.ref, d)
        self.p_a = dv.f64(soa.pa, d)
        self.p_b = dv.f64(soa.pb, d)
        return self

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
        return dv.upload(self.ptrs), dv.f64(self.poses, d)


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


def _vertex_vs_mesh(ga: MeshGeometry, gb: MeshGeometry, threshold: float) -> PairSoA:
    """Best pair per surface vertex of A against B's triangles (collision.py:222-260).

    The all-pairs closest-point scan runs on the GPU (csrc/detect.cu, numpy's
    operation order, bit-exact selection); the host gathers the records of the
    vertices that pass the threshold gate into arrays.
    """
    nv, nt = len(ga.vertex_ids), len(gb.triangles)
    if nv == 0 or nt == 0:
        return PairSoA(0)
    if (ga.dynamic and not ga.deformable) or (gb.dynamic and not gb.deformable):
        raise InvalidAttachmentError("dynamic non-deformable meshes are not supported")
    d = dv.device()
    vids = dv.upload(np.ascontiguousarray(ga.vertex_ids, dtype=np.int64))
    tris = dv.upload(np.ascontiguousarray(gb.triangles, dtype=np.int64))
    pa, pb = _device_points(ga), _device_points(gb)
    work = torch.empty((int(_lib.lib().cnb_detect_work_bytes(nv, nt)) + 7) // 8, dtype=torch.float64, device=d)
    best = torch.empty(nv, dtype=torch.int64, device=d)
    out = torch.empty((nv, 12), dtype=torch.float64, device=d)
    _lib.call("cnb_detect_vertex_mesh", nv, vids.data_ptr(), pa.data_ptr(), nt, tris.data_ptr(), pb.data_ptr(),
              float(threshold), work.data_ptr(), best.data_ptr(), out.data_ptr(), _lib.stream())
    best_h, out_h = best.cpu().numpy(), out.cpu().numpy()
    keep = np.flatnonzero(out_h[:, 11] > 0.0)
    m = len(keep)
    r = PairSoA(m)
    if m == 0:
        return r
    pts_a = np.asarray(ga.points, dtype=np.float64).reshape(-1, 3)
    vid = np.asarray(ga.vertex_ids, dtype=np.int64)[keep]
    t = best_h[keep].astype(np.int64)
    rows = out_h[keep]
    p, cp, nrm = pts_a[vid], rows[:, 5:8], rows[:, 8:11]
    r.obj[:, 0], r.obj[:, 1] = ga.object_id, gb.object_id
    if ga.deformable:
        r.kind[:, 0] = 0
        r.node[:, 0, 0] = vid
        r.w[:, 0, 0] = 1.0
    else:  # kinematic side: the per-point expressions of _mesh_side (same rounding)
        r.kind[:, 0] = 3
        for q in range(m):
            r.local[q, 0] = ga.pose.inverse_apply(p[q])
    if gb.deformable:
        r.kind[:, 1] = 1
        r.node[:, 1] = np.asarray(gb.triangles, dtype=np.int64)[t]
        r.w[:, 1] = rows[:, 2:5]
    else:
        r.kind[:, 1] = 3
        for q in range(m):
            r.local[q, 1] = gb.pose.inverse_apply(cp[q])
            r.lnormal[q] = gb.pose.rotation.T @ nrm[q]
        r.has_ln[:] = 1
    r.pa[:], r.pb[:], r.ref[:] = p, cp, nrm
    r.signed[:] = rows[:, 0]
    r.keys[:] = np.stack([np.full(m, ga.object_id), np.full(m, gb.object_id), vid, t], axis=1)
    return r


def _plane_distances_device(geom: MeshGeometry, plane: PlaneGeometry):
    """float(n @ p - offset) of every surface vertex on the device, bit for bit the
    reference's per-vertex expression (numpy's 3-element dot is an FMA chain,
    csrc/batch.cu plane_distances_kernel); None when the points are host-only."""
    if geom.points_dev is None or len(geom.vertex_ids) == 0:
        return None
    vids = dv.upload(np.ascontiguousarray(geom.vertex_ids, dtype=np.int64))
    pts = _device_points(geom)
    out = dv.empty(len(geom.vertex_ids))
    n = np.asarray(plane.normal, dtype=np.float64)
    _lib.call("cnb_plane_distances", len(geom.vertex_ids), vids.data_ptr(), pts.data_ptr(), float(n[0]),
              float(n[1]), float(n[2]), float(plane.offset), out.data_ptr(), _lib.stream())
    return out.cpu().numpy()


def _vertex_vs_plane(geom: MeshGeometry, plane: PlaneGeometry, threshold: float) -> PairSoA:
    n = plane.normal
    points = np.asarray(geom.points, dtype=np.float64)
    vids_all = np.asarray(geom.vertex_ids, dtype=np.int64)
    d_all = _plane_distances_device(geom, plane)
    if d_all is not None:
        cand = np.arange(len(vids_all))
        exact = d_all
    else:
        # vectorised gate with a margin, then the reference's own expression
        # float(n @ p - offset) per candidate (collision.py:264-270): the kept set
        # and the distances are the reference's bit for bit
        pts = geom.points[geom.vertex_ids]
        approx = pts @ n - plane.offset
        margin = 1e-12 * (np.abs(pts).max(initial=0.0) * np.abs(n).sum() + abs(plane.offset) + 1.0)
        cand = np.flatnonzero(approx <= threshold + margin)
        exact = np.array([float(n @ points[v] - plane.offset) for v in vids_all[cand]])
    keep = exact <= threshold
    m = int(keep.sum())
    r = PairSoA(m)
    if m == 0:
        return r
    if geom.dynamic and not geom.deformable:
        raise InvalidAttachmentError("dynamic non-deformable meshes are not supported")
    vid = vids_all[cand][keep]
    p = points[vid]
    s = exact[keep]
    foot = p - s[:, None] * n
    r.obj[:, 0], r.obj[:, 1] = geom.object_id, plane.object_id
    if geom.deformable:
        r.kind[:, 0] = 0
        r.node[:, 0, 0] = vid
        r.w[:, 0, 0] = 1.0
    else:
        r.kind[:, 0] = 3
        for q in range(m):
            r.local[q, 0] = geom.pose.inverse_apply(p[q])
    r.kind[:, 1] = 4
    r.world[:, 1] = foot
    r.pa[:], r.pb[:] = p, foot
    r.ref[:] = n
    r.signed[:] = s
    r.keys[:] = np.stack([np.full(m, geom.object_id), np.full(m, plane.object_id), vid, np.full(m, -1)], axis=1)
    return r


def _aabbs(meshes):
    """Bounding box of every mesh, once per detection: on the device when the
    points live there (one small read-back), else on the host.  Only a pruning
    gate: it never changes which pairs are found."""
    out = {}
    dev = [g for g in meshes if g.points_dev is not None and len(g.points)]
    if dev:
        mm = torch.stack([torch.cat(torch.aminmax(dv.f64(g.points_dev).reshape(-1, 3), dim=0)) for g in dev])
        mm = mm.cpu().numpy()
        for g, row in zip(dev, mm):
            out[g.object_id] = (row[:3], row[3:])
    for g in meshes:
        if g.object_id not in out:
            pts = np.asarray(g.points, dtype=np.float64).reshape(-1, 3)
            out[g.object_id] = (pts.min(axis=0), pts.max(axis=0)) if len(pts) else (np.full(3, np.inf),
                                                                                  np.full(3, -np.inf))
    return out


def _sphere_vs_plane(sph: SphereGeometry, plane: PlaneGeometry, threshold: float) -> PairSoA:
    """One pair when the sphere is within ``threshold`` of the plane
    (collision.py:290-316): side A the sphere's surface point along -n (a
    body-frame RIGID_LOCAL attachment with its lever), side B its foot on the
    plane (WORLD)."""
    n = plane.normal
    center = np.asarray(sph.center, dtype=np.float64)
    center_dist = float(n @ center - plane.offset)
    signed = center_dist - sph.radius
    r = PairSoA(1 if signed <= threshold else 0)
    if not len(r):
        return r
    surface = center - sph.radius * n
    foot = center - center_dist * n
    r.kind[0] = (2, 4)
    r.obj[0] = (sph.object_id, plane.object_id)
    r.local[0, 0] = sph.pose.inverse_apply(surface)
    r.lever[0] = surface - center
    r.world[0, 1] = foot
    r.pa[0], r.pb[0], r.ref[0] = surface, foot, n
    r.signed[0] = signed
    r.keys[0] = (sph.object_id, plane.object_id, 0, -1)
    return r


def detect_soa(geometries, threshold: float) -> PairSoA:
    """Pairs with signed distance <= threshold in canonical order (collision.py:320-345),
    as arrays."""
    if threshold <= 0:
        raise InvalidAttachmentError(f"threshold must be positive, got {threshold}")
    meshes = [g for g in geometries if isinstance(g, MeshGeometry)]
    planes = [g for g in geometries if isinstance(g, PlaneGeometry)]
    parts = []
    boxes = _aabbs(meshes)
    for ga in meshes:
        for gb in meshes:
            if ga.object_id == gb.object_id or not (ga.dynamic or gb.dynamic):
                continue
            if len(gb.triangles) == 0:
                continue
            lo_a, hi_a = boxes[ga.object_id]
            lo_b, hi_b = boxes[gb.object_id]
            if not (np.all(lo_a - threshold <= hi_b) and np.all(lo_b - threshold <= hi_a)):
                continue
            parts.append(_vertex_vs_mesh(ga, gb, threshold))
        for plane in planes:
            if ga.dynamic:
                parts.append(_vertex_vs_plane(ga, plane, threshold))
    for sph in (g for g in geometries if isinstance(g, SphereGeometry)):
        for plane in planes:
            if sph.dynamic:
                parts.append(_sphere_vs_plane(sph, plane, threshold))
    return PairSoA.concat(parts).sort()


def detect(geometries, threshold: float) -> list:
    """Pairs with signed distance <= threshold in canonical order (collision.py:320-345)."""
    return list(LazyPairs(detect_soa(geometries, threshold)))
