"""Gaussian latitudes (gaussian.py:1-68 of the reference), bit-identical, vectorised.

The returned bits must equal the reference's on the same host: node and target coordinates
decide the noise-level stencil choices.  The reference's arithmetic is
therefore kept op-for-op — the same numpy ufuncs in the same order (Newton on all roots at
once, ``np.arcsin``/``np.degrees``, then the 9-candidate ulp polish keyed by
``|P_2n(sin(radians(c)))|`` with ``math.sin``/``math.radians``) — but the polish, which the
reference evaluates candidate by candidate in a Python loop (45 s at N=1280, SURVEY.md
§6), runs here as one recurrence over all 9·N candidates: elementwise IEEE +,-,*,/ give
the same bits in a vector as on a 0-d array.
"""

from __future__ import annotations

import math

import numpy as np

_MAX_ITER = 100  # gaussian.py:15
_NEWTON_TOL = 1e-15  # gaussian.py:16


def legendre(n: int, x):
    """P_n(x) and P_n'(x) by the three-term recurrence (gaussian.py:19-34)."""
    x = np.asarray(x, dtype=float)
    lo = np.ones_like(x)
    hi = x.copy()
    if n == 0:
        return lo, np.zeros_like(x)
    for k in range(2, n + 1):
        lo, hi = hi, ((2 * k - 1) * x * hi - (k - 1) * lo) / k
    with np.errstate(divide="ignore", invalid="ignore"):
        dp = n * (x * hi - lo) / (x * x - 1.0)
    ends = np.abs(x) == 1.0
    if np.any(ends):
        dp = np.where(ends, x ** (n + 1) * n * (n + 1) / 2.0, dp)
    return hi, dp


def _p_only(n: int, x: np.ndarray) -> np.ndarray:
    lo = np.ones_like(x)
    hi = x.copy()
    if n == 0:
        return lo
    for k in range(2, n + 1):
        lo, hi = hi, ((2 * k - 1) * x * hi - (k - 1) * lo) / k
    return hi


def gaussian_latitudes(n: int) -> np.ndarray:
    """2n Gaussian latitudes in degrees, north to south (gaussian.py:37-62)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    m = 2 * n
    k = np.arange(1, n + 1)
    x = np.cos(np.pi * (k - 0.25) / (m + 0.5))
    for _ in range(_MAX_ITER):
        p, dp = legendre(m, x)
        step = p / dp
        x -= step
        if np.max(np.abs(step)) < _NEWTON_TOL:
            break
    lat = np.degrees(np.arcsin(x))
    # candidate grid: column 0 = lat, then (lo_j, hi_j) for j = 1..4 (gaussian.py:48-54)
    cand = np.empty((n, 9))
    cand[:, 0] = lat
    lo = hi = lat
    for j in range(4):
        lo = np.nextafter(lo, -np.inf)
        hi = np.nextafter(hi, np.inf)
        cand[:, 1 + 2 * j] = lo
        cand[:, 2 + 2 * j] = hi
    # sin(radians(c)) through the same scalar libm calls the reference makes
    s = np.fromiter((math.sin(math.radians(c)) for c in cand.ravel().tolist()), dtype=float,
                    count=cand.size).reshape(cand.shape)
    key = np.abs(_p_only(m, s))
    pick = np.argmin(key, axis=1)  # first minimum, like min(candidates, key=...)
    north = cand[np.arange(n), pick]
    return np.concatenate([north, -north[::-1]])


def legendre_residual(n: int, lats_deg: np.ndarray) -> np.ndarray:
    p, _ = legendre(2 * n, np.sin(np.radians(lats_deg)))
    return np.abs(p)
