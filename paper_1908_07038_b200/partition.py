"""Domain decomposition (partition.py:1-88 of the reference).

``blocks_partition`` cuts the canonical point order into contiguous bands (the only
partitioner the reference has; BASELINE.json's "equal-regions" is absent).
``matching_partition`` slaves a target grid to it: each target point takes the partition
of its nearest master grid point, near-ties (1e-12 relative) going to the smallest global
index.  The nearest-point search is native (sg_matching_partition), using the master's
row structure instead of the reference's cKDTree.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import numpy as np

from . import _native as N
from .errors import TooManyParts
from .grid import Grid

_TIE_RTOL = 1e-12  # partition.py:15


@dataclass(frozen=True)
class Distribution:
    nparts: int
    part_of: np.ndarray  # (npts,) int32

    def __post_init__(self):
        self.part_of.setflags(write=False)

    @property
    def counts(self) -> np.ndarray:
        return np.bincount(self.part_of, minlength=self.nparts)

    def to_dict(self) -> dict:
        return {"nparts": self.nparts, "counts": self.counts.tolist(), "part_of": self.part_of.tolist()}


def blocks_partition(grid: Grid, nparts: int) -> Distribution:
    """Contiguous chunks of the canonical order; the first npts % nparts get one extra."""
    npts = grid.npts
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    if nparts > npts:
        raise TooManyParts(f"{nparts} parts for {npts} points")
    q, r = divmod(npts, nparts)
    bounds = np.arange(nparts + 1, dtype=np.int64) * q + np.minimum(np.arange(nparts + 1), r)
    part_of = (np.searchsorted(bounds, np.arange(npts), side="right") - 1).astype(np.int32)
    return Distribution(nparts=nparts, part_of=part_of)


def nearest_master_points(master: Grid, points: np.ndarray, master_xyz: np.ndarray = None,
                          nthreads: int = 0) -> np.ndarray:
    """Global index of the nearest master grid point of every (m, 3) point, 1e-12 ties ->
    smallest index (PointCloudIndex.query, partition.py:62-75)."""
    pts = np.ascontiguousarray(np.atleast_2d(points), dtype=np.float64)
    mx = np.ascontiguousarray(master.xyz() if master_xyz is None else master_xyz, dtype=np.float64)
    lat = np.ascontiguousarray(master.latitudes, dtype=np.float64)
    nl = np.ascontiguousarray(master.nlons, dtype=np.int64)
    out = np.empty(len(pts), dtype=np.int64)
    N.call("sg_matching_partition", master.nrows, N.ptr(lat), N.ptr(nl), N.ptr(mx), N.ptr(pts),
           len(pts), nthreads, N.ptr(out))
    return out


class PointCloudIndex:
    """Nearest-point index over a grid (partition.py:53-75): same query contract."""

    def __init__(self, grid: Grid):
        self.grid = grid
        self.xyz = grid.xyz()

    def query(self, points: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        idx = nearest_master_points(self.grid, pts, self.xyz)
        return idx, np.linalg.norm(self.xyz[idx] - pts, axis=1)


def nearest_point(index: PointCloudIndex, query_xyz) -> Tuple[int, float]:
    idx, dist = index.query(np.asarray(query_xyz, dtype=float).reshape(1, 3))
    return int(idx[0]), float(dist[0])


def matching_partition(target: Grid, master: Grid, master_dist: Distribution) -> Distribution:
    """Each target point takes the partition of its nearest master point (partition.py:83-88).
    With one partition every point is trivially owned by part 0."""
    if master_dist.nparts == 1:
        return Distribution(nparts=1, part_of=np.zeros(target.npts, dtype=np.int32))
    idx = nearest_master_points(master, target.xyz())
    return Distribution(nparts=master_dist.nparts, part_of=master_dist.part_of[idx].astype(np.int32))


def eq_regions_collars(nparts: int) -> list:
    """Leopardi's recursive zonal equal-area partition of S^2 (the EQ algorithm Atlas's
    EqualRegions partitioner uses): number of regions per zone, north to south — a polar cap
    of 1, collars of n_i, a polar cap of 1."""
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    if nparts == 1:
        return [1]
    if nparts == 2:
        return [1, 1]
    area = 4.0 * np.pi / nparts
    cap = 2.0 * np.arcsin(np.sqrt(1.0 / nparts))  # polar cap colatitude: cap area = one region
    ideal = np.sqrt(area)
    ncollars = max(1, int(round((np.pi - 2.0 * cap) / ideal)))
    fit = (np.pi - 2.0 * cap) / ncollars
    counts, carry = [], 0.0
    for i in range(ncollars):
        top, bot = cap + i * fit, cap + (i + 1) * fit
        ideal_n = 2.0 * np.pi * (np.cos(top) - np.cos(bot)) / area
        n = int(round(ideal_n + carry))
        carry += ideal_n - n
        counts.append(n)
    return [1] + counts + [1]


def equal_regions_partition(grid: Grid, nparts: int) -> Distribution:
    """Equal-regions decomposition (BASELINE.json configs[2] "equal-regions partitioned"; the
    reference has only blocks_partition, so this is an extension — parity unpinned).  Zones
    from eq_regions_collars; the canonical point order (latitude rows north to south) is cut
    into consecutive zone blocks holding exactly the zone's share of points; inside a zone the
    points are ordered by longitude (then canonical order) and cut into its regions.  Part
    sizes equal blocks_partition's (npts // nparts, the first npts % nparts parts one more),
    part ids run north to south, west to east."""
    npts = grid.npts
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    if nparts > npts:
        raise TooManyParts(f"{nparts} parts for {npts} points")
    zones = eq_regions_collars(nparts)
    q, r = divmod(npts, nparts)
    sizes = np.full(nparts, q, np.int64)
    sizes[:r] += 1
    lon = grid.lonlats()[:, 0]
    part_of = np.empty(npts, np.int32)
    p0 = start = 0
    for nz in zones:
        zsizes = sizes[p0:p0 + nz]
        stop = start + int(zsizes.sum())
        idx = np.arange(start, stop)
        order = idx[np.lexsort((idx, lon[start:stop]))]  # by longitude, ties canonical
        bounds = np.concatenate([[0], np.cumsum(zsizes)])
        for k in range(nz):
            part_of[order[bounds[k]:bounds[k + 1]]] = p0 + k
        p0 += nz
        start = stop
    return Distribution(nparts=nparts, part_of=part_of)


PARTITIONERS = {"blocks": blocks_partition, "equal_regions": equal_regions_partition}
