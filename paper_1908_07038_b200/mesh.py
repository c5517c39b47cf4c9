"""Per-partition unstructured mesh (mesh.py:1-420 of the reference), topology native.

``generate_mesh`` returns the reference's ``Mesh`` record.  The integer work — strip-merge
tessellation, element halo levels and BFS, local numbering, connectivity — runs in
``sg_meshgen_create`` (csrc/mesh.cpp, bit-exact by construction, cached serial topology);
the coordinates stay in numpy (``grid.lonlats()[node_global]`` then
``lonlat_to_xyz_array``) so their bits are the reference's (mesh.py:321-330).
Diagnostics (mesh_stats, total_area) and Gmsh export are out of scope.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .errors import InvalidDistribution
from .geometry import lonlat_to_xyz_array
from .grid import Grid
from .partition import Distribution, blocks_partition

TRIANGLE = 3
QUAD = 4


class Shape(enum.Enum):
    TRIANGLE = TRIANGLE
    QUAD = QUAD


@dataclass(frozen=True)
class Connectivity:
    offsets: np.ndarray  # (nelem + 1,) int64
    indices: np.ndarray  # flattened local node indices, int64

    def row(self, e: int) -> np.ndarray:
        return self.indices[self.offsets[e]: self.offsets[e + 1]]

    def __len__(self) -> int:
        return len(self.offsets) - 1


@dataclass(frozen=True)
class Node:
    global_index: int
    lon: float
    lat: float
    partition: int
    remote_index: int
    ghost: bool
    halo_level: int


@dataclass(frozen=True)
class Element:
    shape: Shape
    nodes: Tuple[int, ...]
    halo_level: int


@dataclass
class Mesh:
    grid: Grid
    partition_id: int
    nparts: int
    halo_depth: int
    include_pole: bool
    node_global: np.ndarray  # int64
    node_lonlat: np.ndarray  # (n, 2)
    node_xyz: np.ndarray  # (n, 3)
    node_part: np.ndarray  # int32
    node_remote: np.ndarray  # int64, row on the owning partition
    node_ghost: np.ndarray  # bool
    node_halo: np.ndarray  # int16
    element_connectivity: Connectivity
    elem_halo: np.ndarray  # int16
    elem_serial_id: np.ndarray  # int64

    @property
    def nb_nodes(self) -> int:
        return len(self.node_global)

    @property
    def nb_owned_nodes(self) -> int:
        return int(np.count_nonzero(~self.node_ghost))

    @property
    def nb_elements(self) -> int:
        return len(self.element_connectivity)

    def node(self, i: int) -> Node:
        return Node(int(self.node_global[i]), float(self.node_lonlat[i, 0]), float(self.node_lonlat[i, 1]),
                    int(self.node_part[i]), int(self.node_remote[i]), bool(self.node_ghost[i]),
                    int(self.node_halo[i]))

    def element(self, e: int) -> Element:
        row = self.element_connectivity.row(e)
        return Element(Shape.TRIANGLE if len(row) == 3 else Shape.QUAD, tuple(int(i) for i in row),
                       int(self.elem_halo[e]))

    def elements_nodes(self) -> List[np.ndarray]:
        return [self.element_connectivity.row(e) for e in range(self.nb_elements)]


def _lonlat_with_poles(grid: Grid, include_pole: bool) -> np.ndarray:
    ll = grid.lonlats()
    if include_pole:
        ll = np.vstack([ll, [[0.0, 90.0], [0.0, -90.0]]])
    return ll


def generate_mesh(grid: Grid, dist: Distribution, part: int = 0, halo: int = 0,
                  include_pole: bool = False) -> Mesh:
    """Mesh of partition ``part`` with ``halo`` layers of ghost elements (mesh.py:229-338)."""
    if len(dist.part_of) != grid.npts:
        raise InvalidDistribution(f"distribution sized {len(dist.part_of)} for a grid of {grid.npts} points")
    if not 0 <= part < dist.nparts:
        raise ValueError(f"partition {part} not in [0, {dist.nparts})")
    nlons = np.ascontiguousarray(grid.nlons, dtype=np.int64)
    part_of = np.ascontiguousarray(dist.part_of, dtype=np.int32)
    h = C.c_uint64(0)
    nn, no, ne, ni = (C.c_int64(0) for _ in range(4))
    N.call("sg_meshgen_create", grid.nrows, N.ptr(nlons), int(bool(include_pole)), N.ptr(part_of),
           grid.npts, dist.nparts, part, halo, N.ref(h), N.ref(nn), N.ref(no), N.ref(ne), N.ref(ni))
    handle = N.Handle(h.value)
    try:
        node_global = np.empty(nn.value, np.int64)
        node_part = np.empty(nn.value, np.int32)
        node_remote = np.empty(nn.value, np.int64)
        node_ghost = np.empty(nn.value, np.bool_)
        node_halo = np.empty(nn.value, np.int16)
        offsets = np.empty(ne.value + 1, np.int64)
        indices = np.empty(ni.value, np.int64)
        elem_halo = np.empty(ne.value, np.int16)
        serial = np.empty(ne.value, np.int64)
        N.call("sg_meshgen_fetch", handle.handle, N.ptr(node_global), N.ptr(node_part), N.ptr(node_remote),
               N.ptr(node_ghost), N.ptr(node_halo), N.ptr(offsets), N.ptr(indices), N.ptr(elem_halo),
               N.ptr(serial))
    finally:
        handle.close()
    lonlat = _lonlat_with_poles(grid, include_pole)[node_global]
    return Mesh(
        grid=grid, partition_id=part, nparts=dist.nparts, halo_depth=halo, include_pole=include_pole,
        node_global=node_global, node_lonlat=lonlat,
        node_xyz=lonlat_to_xyz_array(lonlat[:, 0], lonlat[:, 1]),
        node_part=node_part, node_remote=node_remote, node_ghost=node_ghost, node_halo=node_halo,
        element_connectivity=Connectivity(offsets=offsets, indices=indices),
        elem_halo=elem_halo, elem_serial_id=serial,
    )


def split_quad(row: np.ndarray) -> List[np.ndarray]:
    """Quad -> two triangles by the diagonal at the lowest local index (mesh.py:395-403)."""
    m = int(np.argmin(row))
    c = [int(row[(m + k) % 4]) for k in range(4)]
    return [np.asarray(c[:3], dtype=np.int64), np.asarray([c[0], c[2], c[3]], dtype=np.int64)]


def element_triangles(mesh: Mesh, e: int) -> List[np.ndarray]:
    row = mesh.element_connectivity.row(e)
    return [np.asarray(row, dtype=np.int64)] if len(row) == 3 else split_quad(row)


# -- serial topology and mesh diagnostics (mesh.py:134-140, 174-226, 344-420 of the reference) --

@dataclass
class SerialTopology:
    nnodes: int                    # grid.npts (+2 with poles)
    elem_nodes: List[np.ndarray]   # global node ids per element, serial order
    node_lonlat: np.ndarray
    north_pole: Optional[int]
    south_pole: Optional[int]


def serial_topology(grid: Grid, include_pole: bool) -> SerialTopology:
    """The global element sweep (mesh.py:174-226): the one-partition, halo-0 mesh of the
    native generator, whose local numbering is the global one."""
    m = generate_mesh(grid, blocks_partition(grid, 1), 0, halo=0, include_pole=include_pole)
    conn = m.element_connectivity
    gidx = m.node_global[conn.indices]
    elem_nodes = [gidx[conn.offsets[e]:conn.offsets[e + 1]] for e in range(len(conn))]
    order = np.argsort(m.elem_serial_id, kind="stable")
    npts = grid.npts
    return SerialTopology(
        nnodes=npts + (2 if include_pole else 0), elem_nodes=[elem_nodes[e] for e in order],
        node_lonlat=_lonlat_with_poles(grid, include_pole),
        north_pole=npts if include_pole else None, south_pole=npts + 1 if include_pole else None)


def _edges(mesh: Mesh) -> np.ndarray:
    """Unique undirected element sides as sorted (i, j) pairs."""
    off, idx = mesh.element_connectivity.offsets, mesh.element_connectivity.indices
    k = np.diff(off)
    pos = np.arange(len(idx), dtype=np.int64)
    first = np.repeat(off[:-1], k)
    nxt = np.where(pos + 1 < np.repeat(off[1:], k), pos + 1, first)
    a, b = idx, idx[nxt]
    pairs = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1)
    return np.unique(pairs, axis=0) if len(pairs) else pairs


def mesh_stats(mesh: Mesh) -> dict:
    """V, E (unique sides), F, Euler characteristic and owned counts (mesh.py:355-375); an
    element is owned by the partition owning its lowest-partition node."""
    off, idx = mesh.element_connectivity.offsets, mesh.element_connectivity.indices
    v, f = mesh.nb_nodes, mesh.nb_elements
    e = len(_edges(mesh))
    owned = int((np.minimum.reduceat(mesh.node_part[idx], off[:-1]) == mesh.partition_id).sum()) if f else 0
    return {"V": v, "E": e, "F": f, "chi": v - e + f, "owned_nodes": mesh.nb_owned_nodes, "owned_elements": owned}


def total_area(mesh: Mesh) -> float:
    """Sum of spherical triangle areas over the split elements, L'Huilier's theorem
    (mesh.py:378-420), vectorised over all triangles."""
    tris = [t for e in range(mesh.nb_elements) for t in element_triangles(mesh, e)]
    if not tris:
        return 0.0
    t = np.asarray(tris, dtype=np.int64)
    a, b, c = (mesh.node_xyz[t[:, i]] for i in range(3))

    def angle(u, w):
        return np.arctan2(np.linalg.norm(np.cross(u, w), axis=1), np.einsum("ij,ij->i", u, w))

    sa, sb, sc = angle(b, c), angle(c, a), angle(a, b)
    s = 0.5 * (sa + sb + sc)
    x = np.tan(0.5 * s) * np.tan(0.5 * (s - sa)) * np.tan(0.5 * (s - sb)) * np.tan(0.5 * (s - sc))
    return float(np.sum(4.0 * np.arctan(np.sqrt(np.maximum(x, 0.0)))))
