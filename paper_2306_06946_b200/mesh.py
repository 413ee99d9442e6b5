"""Tetrahedral meshes: container, procedural grids, surface extraction, ASCII I/O.

Host-side preprocessing (outside the hot path).  The integer conventions are
parity-relevant and follow the reference (/root/reference/pkg/src/contactnewton/mesh.py):

* surface triangles are the tet faces seen once, wound outward with the face
  table of mesh.py:106, sorted by their oriented node tuple (mesh.py:109-122);
  a contact's ``element_id`` indexes that sorted list;
* ``box_mesh`` is the 6-tet Kuhn split with x-fastest node numbering
  (mesh.py:59-101), used by scene files;
* ``five_tet_grid`` is the 5-tets-per-hex grid of the BASELINE configs
  (not in the reference: SURVEY.md §9 #3), alternating the two mirror
  patterns by cell parity so faces conform, every tet positively oriented.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DegenerateTetError, ParseError


@dataclass
class TetMesh:
    nodes: np.ndarray  # (n, 3) float64, metres
    tets: np.ndarray  # (m, 4) int64

    def __post_init__(self):
        self.nodes = np.asarray(self.nodes, dtype=np.float64).reshape(-1, 3)
        self.tets = np.asarray(self.tets, dtype=np.int64).reshape(-1, 4)
        if self.tets.size and (self.tets.min() < 0 or self.tets.max() >= len(self.nodes)):
            raise ParseError("tet indices out of range")

    @property
    def n_nodes(self) -> int:
        return len(self.nodes)

    @property
    def n_tets(self) -> int:
        return len(self.tets)


def tet_volumes(nodes: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """Signed volumes (positive = correctly oriented)."""
    p = nodes[tets]
    e1, e2, e3 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]
    return np.einsum("ij,ij->i", np.cross(e1, e2), e3) / 6.0


def check_positive_volumes(mesh: TetMesh, where: str = "mesh") -> np.ndarray:
    vols = tet_volumes(mesh.nodes, mesh.tets)
    if vols.size and vols.min() <= 0.0:
        k = int(np.argmin(vols))
        raise DegenerateTetError(f"{where}: tet {k} has non-positive volume {vols[k]:.3e}")
    return vols


def _grid_nodes(shape, spacing, origin):
    nx, ny, nz = shape
    xs = origin[0] + spacing[0] * np.arange(nx)
    ys = origin[1] + spacing[1] * np.arange(ny)
    zs = origin[2] + spacing[2] * np.arange(nz)
    gz, gy, gx = np.meshgrid(zs, ys, xs, indexing="ij")
    return np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])


def _cell_corners(nx, ny, nz):
    """(cells, 8) node ids of each hex, corner bit pattern x + 2y + 4z."""
    i, j, k = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), np.arange(nz - 1), indexing="ij")
    i, j, k = (a.transpose(2, 1, 0).ravel() for a in (i, j, k))  # x fastest, then y, then z
    bits = np.arange(8)
    ci = i[:, None] + (bits & 1)
    cj = j[:, None] + ((bits >> 1) & 1)
    ck = k[:, None] + ((bits >> 2) & 1)
    return ci + nx * (cj + ny * ck), (i + j + k) & 1


_KUHN = np.array([(0, 1, 3, 7), (0, 3, 2, 7), (0, 2, 6, 7), (0, 6, 4, 7), (0, 4, 5, 7), (0, 5, 1, 7)])
# 5-tet split: one central tet plus four corner tets; the odd-parity pattern
# is the mirror image so neighbouring cells share face diagonals.
_FIVE_EVEN = np.array([(1, 2, 4, 7), (0, 1, 2, 4), (3, 1, 7, 2), (5, 1, 4, 7), (6, 2, 7, 4)])
_FIVE_ODD = np.array([(0, 3, 5, 6), (1, 0, 5, 3), (2, 0, 3, 6), (4, 0, 6, 5), (7, 3, 6, 5)])


def _orient(nodes, tets):
    vol = tet_volumes(nodes, tets)
    flip = vol < 0
    tets = tets.copy()
    tets[flip, 2], tets[flip, 3] = tets[flip, 3].copy(), tets[flip, 2].copy()
    return tets


def box_mesh(size, divisions, center=(0.0, 0.0, 0.0)) -> TetMesh:
    """Axis-aligned box, Kuhn 6-tet cells, (nx+1)(ny+1)(nz+1) nodes, x fastest."""
    size = np.asarray(size, dtype=np.float64)
    center = np.asarray(center, dtype=np.float64)
    nx, ny, nz = (int(d) for d in divisions)
    if min(nx, ny, nz) < 1 or np.any(size <= 0):
        raise ParseError(f"invalid box mesh: size={size.tolist()}, divisions={divisions}")
    axes = [np.linspace(-0.5, 0.5, d + 1) * s + c for d, s, c in zip((nx, ny, nz), size, center)]
    gz, gy, gx = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    nodes = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    corners, _ = _cell_corners(nx + 1, ny + 1, nz + 1)
    tets = corners[:, _KUHN].reshape(-1, 4)
    mesh = TetMesh(nodes, tets)
    check_positive_volumes(mesh, "box_mesh")
    return mesh


def five_tet_grid(shape, spacing=0.01, origin=(0.0, 0.0, 0.0)) -> TetMesh:
    """Hexahedral node grid of ``shape`` = (nx, ny, nz) NODES, 5 tets per hex."""
    nx, ny, nz = (int(s) for s in shape)
    if min(nx, ny, nz) < 2:
        raise ParseError(f"five_tet_grid needs >= 2 nodes per axis, got {shape}")
    sp_ = np.broadcast_to(np.asarray(spacing, dtype=np.float64), (3,))
    nodes = _grid_nodes((nx, ny, nz), sp_, np.asarray(origin, dtype=np.float64))
    corners, parity = _cell_corners(nx, ny, nz)
    tets = np.where(parity[:, None, None] == 0, corners[:, _FIVE_EVEN], corners[:, _FIVE_ODD])
    tets = _orient(nodes, tets.reshape(-1, 4))
    mesh = TetMesh(nodes, tets)
    check_positive_volumes(mesh, "five_tet_grid")
    return mesh


_TET_FACES = np.array([(0, 2, 1), (0, 1, 3), (0, 3, 2), (1, 2, 3)])


def surface_triangles(mesh_or_tets) -> np.ndarray:
    """Outward boundary faces in sorted oriented-tuple order (element ids)."""
    tets = mesh_or_tets.tets if isinstance(mesh_or_tets, TetMesh) else np.asarray(mesh_or_tets)
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    if len(tets) == 0:
        return np.zeros((0, 3), dtype=np.int64)
    faces = tets[:, _TET_FACES].reshape(-1, 3)
    key = np.sort(faces, axis=1)
    n = int(key.max()) + 1
    code = (key[:, 0] * n + key[:, 1]) * n + key[:, 2]
    uniq, inverse, counts = np.unique(code, return_inverse=True, return_counts=True)
    once = faces[counts[inverse] == 1]
    order = np.lexsort((once[:, 2], once[:, 1], once[:, 0]))
    return once[order]


def surface_vertices(triangles: np.ndarray) -> np.ndarray:
    return np.unique(np.asarray(triangles).ravel())


def save_mesh(mesh: TetMesh, path) -> None:
    with open(path, "w") as fh:
        fh.write(f"nodes {mesh.n_nodes}\n")
        for x, y, z in mesh.nodes:
            fh.write(f"{float(x)!r} {float(y)!r} {float(z)!r}\n")
        fh.write(f"tets {mesh.n_tets}\n")
        for t in mesh.tets:
            fh.write(f"{t[0]} {t[1]} {t[2]} {t[3]}\n")


def load_mesh(path) -> TetMesh:
    """ASCII format: 'nodes N' + N coordinate lines, 'tets M' + M index lines; '#' comments."""
    section, nodes, tets = None, [], []
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            try:
                if tok[0] in ("nodes", "tets"):
                    section = tok[0]
                    int(tok[1])
                elif section is None:
                    raise ValueError("data before section header")
                elif section == "nodes":
                    if len(tok) != 3:
                        raise ValueError("node line needs 3 coordinates")
                    nodes.append([float(v) for v in tok])
                else:
                    if len(tok) != 4:
                        raise ValueError("tet line needs 4 indices")
                    tets.append([int(v) for v in tok])
            except (ValueError, IndexError) as exc:
                raise ParseError(f"{path}:{lineno}: {exc}") from exc
    return TetMesh(np.array(nodes, dtype=np.float64).reshape(-1, 3),
                   np.array(tets, dtype=np.int64).reshape(-1, 4))
