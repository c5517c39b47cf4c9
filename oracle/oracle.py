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
