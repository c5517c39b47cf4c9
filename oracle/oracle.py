"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatements of the reference's hot-path functions, each citing the reference
file:line it follows (paths relative to /root/reference/pkg/src/spheregrid/).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from typing import Dict, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "liblocate_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


def _c():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.oracle_locate.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_void_p, C.c_void_p]
        _lib.oracle_locate.restype = C.c_int
        _lib.oracle_locate_knn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                           C.c_int64, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _lib.oracle_locate_knn.restype = C.c_int
        _lib.oracle_dgesv3.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        _lib.oracle_dgesv3.restype = C.c_int64
    return _lib


def locate(node_xyz: np.ndarray, conn_off: np.ndarray, conn_idx: np.ndarray, points: np.ndarray
           ) -> Tuple[np.ndarray, np.ndarray]:
    """MeshLocator.locate for each point (interp.py:102-117): element id (-1 NotLocated,
    -2 DegenerateTriangle) and local corner triple."""
    xyz = np.ascontiguousarray(node_xyz, np.float64)
    off = np.ascontiguousarray(conn_off, np.int64)
    idx = np.ascontiguousarray(conn_idx, np.int64)
    pts = np.ascontiguousarray(np.atleast_2d(points), np.float64)
    elem = np.empty(len(pts), np.int64)
    corners = np.empty((len(pts), 3), np.int64)
    _c().oracle_locate(xyz.ctypes.data, len(xyz), off.ctypes.data, idx.ctypes.data, len(off) - 1,
                       pts.ctypes.data, len(pts), elem.ctypes.data, corners.ctypes.data)
    return elem, corners


def barycentric_weights(a, b, c, p) -> np.ndarray:
    """interp.py:61-71: solve [a b c] w = p (LAPACK dgesv via numpy), then w / sum(w)."""
    w = np.linalg.solve(np.column_stack([a, b, c]), p)
    return w / w.sum()


def build_remap(node_xyz, conn_off, conn_idx, target_xyz) -> Dict[str, np.ndarray]:
    """build_remap's per-target loop (interp.py:175-194) without fallback: nodes, weights,
    scale; rows that are not located get nodes -1."""
    elem, corners = locate(node_xyz, conn_off, conn_idx, target_xyz)
    m = len(target_xyz)
    weights = np.zeros((m, 3))
    scale = np.ones(m)
    for k in range(m):
        if elem[k] < 0:
            continue
        a, b, c = (node_xyz[i] for i in corners[k])
        w = barycentric_weights(a, b, c, target_xyz[k])
        weights[k] = w
        scale[k] = float(w @ np.column_stack([a, b, c]).T @ target_xyz[k])
    return {"elem": elem, "nodes": corners, "weights": weights, "scale": scale}


def apply_remap(nodes: np.ndarray, weights: np.ndarray, src: np.ndarray) -> np.ndarray:
    """interp.py:219-223, the same numpy expression (each op separately rounded)."""
    return (weights[:, 0:1] * src[nodes[:, 0]] + weights[:, 1:2] * src[nodes[:, 1]]
            + weights[:, 2:3] * src[nodes[:, 2]])


def halo_payloads(send: Dict[int, np.ndarray], host: np.ndarray) -> Dict[int, bytes]:
    """functionspace.py:113-114: one payload per peer, f.host[send[peer]].tobytes()."""
    return {p: host[send[p]].tobytes() for p in sorted(send)}


def halo_unpack(recv: Dict[int, np.ndarray], host: np.ndarray, payloads: Dict[int, bytes]) -> np.ndarray:
    """functionspace.py:115-117."""
    out = host.copy()
    for p in sorted(recv):
        out[recv[p]] = np.frombuffer(payloads[p], dtype=host.dtype).reshape(len(recv[p]), host.shape[1])
    return out


def nearest_points(master_xyz: np.ndarray, points: np.ndarray, chunk: int = 256) -> np.ndarray:
    """PointCloudIndex.query (partition.py:62-75) by brute force: nearest by
    np.linalg.norm, ties within 1e-12 relative -> smallest index."""
    out = np.empty(len(points), np.int64)
    for s in range(0, len(points), chunk):
        p = points[s:s + chunk]
        d = np.linalg.norm(master_xyz[None, :, :] - p[:, None, :], axis=2)
        best = d.min(axis=1, keepdims=True)
        ok = d <= best * (1.0 + 1e-12)
        out[s:s + chunk] = np.argmax(ok, axis=1)
    return out


def blocks_partition(npts: int, nparts: int) -> np.ndarray:
    """partition.py:38-50."""
    base, extra = divmod(npts, nparts)
    sizes = np.full(nparts, base, np.int64)
    sizes[:extra] += 1
    return np.repeat(np.arange(nparts, dtype=np.int32), sizes)


def legendre_p(n: int, x: float) -> float:
    """gaussian.py:19-34, scalar."""
    p_prev, p = 1.0, x
    for k in range(2, n + 1):
        p_prev, p = p, ((2 * k - 1) * x * p - (k - 1) * p_prev) / k
    return p


def gaussian_latitudes(n: int) -> np.ndarray:
    """gaussian.py:37-62 restated with numpy ufuncs on the same vectors (the arcsin bits
    are numpy's)."""
    m = 2 * n
    k = np.arange(1, n + 1)
    x = np.cos(np.pi * (k - 0.25) / (m + 0.5))
    for _ in range(100):
        p_prev, p = np.ones_like(x), x.copy()
        for j in range(2, m + 1):
            p_prev, p = p, ((2 * j - 1) * x * p - (j - 1) * p_prev) / j
        dp = m * (x * p - p_prev) / (x * x - 1.0)
        dx = p / dp
        x -= dx
        if np.max(np.abs(dx)) < 1e-15:
            break
    lat = np.degrees(np.arcsin(x))
    out = []
    for v in lat:
        cands = [v]
        lo = hi = v
        for _ in range(4):
            lo, hi = np.nextafter(lo, -np.inf), np.nextafter(hi, np.inf)
            cands += [lo, hi]
        out.append(min(cands, key=lambda c: abs(legendre_p(m, math.sin(math.radians(c))))))
    north = np.array(out)
    return np.concatenate([north, -north[::-1]])


def apply_remap_k(nodes: np.ndarray, weights: np.ndarray, src: np.ndarray) -> np.ndarray:
    """k-point apply, summed left to right: ((w0*s0 + w1*s1) + w2*s2) [+ w3*s3]."""
    out = weights[:, 0:1] * src[nodes[:, 0]] + weights[:, 1:2] * src[nodes[:, 1]]
    for k in range(2, nodes.shape[1]):
        out = out + weights[:, k:k + 1] * src[nodes[:, k]]
    return out


def bilinear_stencil(lat: np.ndarray, nlons: np.ndarray, lonlat: np.ndarray, has_poles: bool):
    """Structured-bilinear stencils — NOT a reference function (the reference has no bilinear
    method; parity unpinned).  CPU restatement of the definition in
    paper_1908_07038_b200/csrc/bilinear.cu: returns (global nodes (m, 4), weights (m, 4),
    located (m,))."""
    lat = np.asarray(lat, float)
    nlons = np.asarray(nlons, np.int64)
    off = np.concatenate([[0], np.cumsum(nlons)])
    npts = int(off[-1])
    lam, phi = lonlat[:, 0], lonlat[:, 1]
    m = len(lonlat)
    nodes = np.zeros((m, 4), np.int64)
    w = np.zeros((m, 4))
    ok = np.ones(m, bool)

    def row_pair(j, lam_):
        n = nlons[j]
        x = (lam_ * n.astype(float)) / 360.0
        i = np.clip(np.floor(x).astype(np.int64), 0, n - 1)
        a = x - i.astype(float)
        return off[j] + i, off[j] + (i + 1) % n, a

    north, south = phi > lat[0], phi < lat[-1]
    inner = ~(north | south)
    j = np.searchsorted(-lat, -phi[inner], side="right") - 1
    j = np.minimum(j, len(lat) - 2)
    beta = (lat[j] - phi[inner]) / (lat[j] - lat[j + 1])
    ia, ib, a0 = row_pair(j, lam[inner])
    ic, id_, a1 = row_pair(j + 1, lam[inner])
    ob = 1.0 - beta
    nodes[inner] = np.stack([ia, ib, ic, id_], 1)
    w[inner] = np.stack([ob * (1.0 - a0), ob * a0, beta * (1.0 - a1), beta * a1], 1)
    for cap, jj, pole in ((north, 0, npts), (south, len(lat) - 1, npts + 1)):
        if not cap.any():
            continue
        if not has_poles:
            ok[cap] = False
            continue
        p = phi[cap]
        beta = (90.0 - p) / (90.0 - lat[0]) if jj == 0 else (p + 90.0) / (lat[jj] + 90.0)
        ia, ib, a = row_pair(np.full(cap.sum(), jj), lam[cap])
        nodes[cap] = np.stack([np.full(cap.sum(), pole), ia, ib, np.full(cap.sum(), pole)], 1)
        w[cap] = np.stack([1.0 - beta, beta * (1.0 - a), beta * a, np.zeros(cap.sum())], 1)
    return nodes, w, ok


def locate_kdtree(node_xyz, conn_off, conn_idx, points, workers: int = -1):
    """MeshLocator.locate at scale (interp.py:90-117): candidates from the reference's own
    scipy cKDTree (k = 8, then 32 for points not located, interp.py:106), scored in C with
    the reference's arithmetic and first-wins order.  Returns (elem, corners) like locate()."""
    from scipy.spatial import cKDTree

    xyz = np.ascontiguousarray(node_xyz, np.float64)
    off = np.ascontiguousarray(conn_off, np.int64)
    idx = np.ascontiguousarray(conn_idx, np.int64)
    pts = np.ascontiguousarray(np.atleast_2d(points), np.float64)
    tree = cKDTree(xyz)
    elem = np.full(len(pts), -1, np.int64)
    corners = np.full((len(pts), 3), -1, np.int64)
    todo = np.arange(len(pts))
    for k in (8, 32):
        if len(todo) == 0:
            break
        kk = min(k, len(xyz))
        _, nn = tree.query(pts[todo], k=kk, workers=workers)
        nn = np.ascontiguousarray(np.asarray(nn).reshape(len(todo), kk), np.int64)
        sub = np.ascontiguousarray(pts[todo])
        e = np.empty(len(todo), np.int64)
        c = np.empty((len(todo), 3), np.int64)
        _c().oracle_locate_knn(xyz.ctypes.data, len(xyz), off.ctypes.data, idx.ctypes.data, len(off) - 1,
                               sub.ctypes.data, len(sub), nn.ctypes.data, kk, e.ctypes.data, c.ctypes.data)
        elem[todo], corners[todo] = e, c
        todo = todo[e == -1]
    return elem, corners


def dgesv3_restated(M: np.ndarray, p: np.ndarray) -> np.ndarray:
    """np.linalg.solve for (m, 3, 3) systems restated as numpy's OpenBLAS dgesv evaluates it
    (locate_oracle.c oracle_dgesv3; the checker of csrc/locate.cu lu_solve3, interp.py:65)."""
    M = np.ascontiguousarray(M, np.float64)
    p = np.ascontiguousarray(p, np.float64)
    x = np.empty((len(M), 3))
    if _c().oracle_dgesv3(M.ctypes.data, p.ctypes.data, x.ctypes.data, len(M)):
        raise np.linalg.LinAlgError("singular matrix")
    return x


def barycentric_weights_batched(xyz, corners, points):
    """barycentric_weights (interp.py:61-71) for many points: one batched LAPACK solve of the
    (m, 3, 3) vertex matrices, then w / sum(w).  Weights agree with the per-point calls to
    ~1e-16 (same dgesv; batching may change the BLAS kernel)."""
    M = np.stack([xyz[corners[:, 0]], xyz[corners[:, 1]], xyz[corners[:, 2]]], axis=2)
    w = np.linalg.solve(M, points[:, :, None])[:, :, 0]
    return w / w.sum(axis=1, keepdims=True)


_MIX = (np.uint64(0x9E3779B97F4A7C15), np.uint64(0xC2B2AE3D27D4EB4F), np.uint64(0xBF58476D1CE4E5B9),
        np.uint64(0x94D049BB133111EB))


def checksum_partial(gids: np.ndarray, values: np.ndarray) -> int:
    """functionspace.py:233-248 restated: wrapping u64 sum over (point, level) of
    splitmix64_finalizer(gid*G + (level+1)*Lv ^ value_bits)."""
    gamma, lev, m1, m2 = _MIX
    bits = values.view(np.uint64) if values.dtype.itemsize == 8 else values.view(np.uint32).astype(np.uint64)
    levels = np.arange(values.shape[1], dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (gids.astype(np.uint64)[:, None] * gamma + (levels[None, :] + np.uint64(1)) * lev) ^ bits
        x ^= x >> np.uint64(30)
        x *= m1
        x ^= x >> np.uint64(27)
        x *= m2
        x ^= x >> np.uint64(31)
        return int(np.sum(x, dtype=np.uint64))
