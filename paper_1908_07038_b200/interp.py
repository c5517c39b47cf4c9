"""Linear element remapping on the GPU (interp.py:1-235 of the reference).

``build_remap`` and ``apply_remap`` keep the reference's signatures, return types,
exceptions and state transitions; the work runs in libsgb200:

* ``MeshLocator`` uploads the mesh once and builds the device search structure
  (sg_locator_create); ``locate`` is batched (sg_locator_locate).
* ``build_remap`` locates every owned target, computes gnomonic barycentric weights and the
  projection scale in one kernel (sg_remap_build) and keeps the device stencil attached to
  the returned ``InterpolationWeights`` for ``apply_remap``.  Zero messages (interp.py:9-11).
* ``apply_remap`` is the multi-level SpMM kernel (sg_remap_apply), bitwise equal to the
  numpy expression of interp.py:219-223, with the reference's contract for every field
  state (result in ``target.host``; SYNCED -> HOST_DIRTY): SYNCED sources are read from
  HBM, the others are staged from the host.  ``apply_remap_device_fields`` is the opt-in
  HBM-only entry point (target left DEVICE_DIRTY).
* ``Interpolation(source_fs, target, target_dist, ctx).execute(src, tgt)`` is the Atlas
  spelling: build once, apply per call.

The module-level constants are the reference's (interp.py:29-31).  The kNN candidate
widths are kept for API parity; the device search scores a superset of the kNN candidates
and applies the reference's tie rule explicitly (see csrc/locate.cu).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .device import DeviceArray, current_device
from .errors import DegenerateTriangle, NoDevice, NotLocated, ShapeMismatch, SpheregridError, StaleDevice
from .field import Field, MemoryState
from .functionspace import NodeColumns
from .grid import Grid
from .mesh import Mesh
from .partition import Distribution

CONTAIN_EPS = 1e-12
_KNN_FIRST = 8
_KNN_WIDE = 32

APPLY_DEFAULT, APPLY_WARP, APPLY_BULK = 0, 1, 2
# host-buffer execute path used by apply_remap on host-resident fields (see execute_host)
HOST_EXECUTE_MODE = "auto"
HOST_EXECUTE_CHUNKS = 0  # 0: min(64, targets / 16384)
HOST_EXECUTE_DIRECT_PERIOD = 0  # compact mode: every n-th chunk copied directly (0: none)


@dataclass(frozen=True)
class SphericalTriangle:
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray

    def __post_init__(self):
        vol = float(np.dot(np.cross(self.a, self.b), self.c))
        if abs(vol) <= 1e-15:
            raise DegenerateTriangle(f"triple product {vol}")


def signed_tests(tri: SphericalTriangle, p: np.ndarray) -> Tuple[float, float, float]:
    """Edge-plane tests (interp.py:46-51); scalar host helper, not on the hot path."""
    return tuple(float(np.dot(np.cross(u, v), p)) for u, v in ((tri.a, tri.b), (tri.b, tri.c), (tri.c, tri.a)))


def contains(tri: SphericalTriangle, p: np.ndarray, eps: float = CONTAIN_EPS) -> bool:
    return all(t >= -eps for t in signed_tests(tri, p))


def barycentric_weights(tri: SphericalTriangle, p: np.ndarray) -> np.ndarray:
    """Gnomonic weights of one point (interp.py:61-71); scalar host helper."""
    m = np.column_stack([tri.a, tri.b, tri.c])
    try:
        w = np.linalg.solve(m, p)
    except np.linalg.LinAlgError:
        raise DegenerateTriangle("singular vertex matrix") from None
    s = w.sum()
    if s == 0.0:
        raise DegenerateTriangle("projection plane through the origin")
    return w / s


class MeshLocator:
    """Device point location in a mesh (interp.py:74-117)."""

    def __init__(self, mesh: Mesh, device: Optional[int] = None):
        self.mesh = mesh
        self.device = current_device() if device is None else device
        conn = mesh.element_connectivity
        xyz = np.ascontiguousarray(mesh.node_xyz, dtype=np.float64)
        off = np.ascontiguousarray(conn.offsets, dtype=np.int64)
        idx = np.ascontiguousarray(conn.indices, dtype=np.int64)
        h = C.c_uint64(0)
        N.call("sg_locator_create", self.device, N.ptr(xyz), mesh.nb_nodes, N.ptr(off), N.ptr(idx),
               mesh.nb_elements, N.ref(h))
        self._h = N.Handle(h.value)

    @property
    def handle(self) -> int:
        return self._h.handle

    def stats(self) -> dict:
        nt, nb, ne, band = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        N.call("sg_locator_stats", self.handle, N.ref(nt), N.ref(nb), N.ref(ne), N.ref(band))
        return {"triangles": nt.value, "bins": nb.value, "entries": ne.value, "band_rad": band.value}

    def locate_many(self, points: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        """(m, 3) points -> (element ids (m,), corner triples (m, 3)); element -1 where not
        located, -2 where the reference raises DegenerateTriangle (a degenerate triangle among
        its kNN candidates, interp.py:34-43), -3 undecidable."""
        pts = np.ascontiguousarray(np.atleast_2d(points), dtype=np.float64)
        elem = np.empty(len(pts), np.int64)
        corners = np.empty((len(pts), 3), np.int64)
        N.call("sg_locator_locate", self.handle, N.ptr(pts), len(pts), N.ptr(elem), N.ptr(corners))
        return elem, corners

    def locate(self, p: np.ndarray):
        """-> (element id, triangle, local corner indices) or NotLocated (interp.py:102-117)."""
        elem, corners = self.locate_many(np.asarray(p, dtype=float).reshape(1, 3))
        if elem[0] == -2:
            raise DegenerateTriangle("degenerate candidate triangle")  # interp.py:40-43
        if elem[0] == -3:
            raise SpheregridError("too many overlapping candidate triangles to decide")
        if elem[0] < 0:
            raise NotLocated("point not contained in any candidate element")
        xyz = self.mesh.node_xyz
        c = corners[0]
        return int(elem[0]), SphericalTriangle(xyz[c[0]], xyz[c[1]], xyz[c[2]]), c


@dataclass
class InterpolationWeights:
    """Per owned target: 3 local source nodes and weights (interp.py:120-151); ``stencil``
    holds the device copy used by apply_remap."""

    target_global: np.ndarray
    nodes: np.ndarray
    weights: np.ndarray
    fallback: np.ndarray
    source_nnodes: int = 0
    source_global: Optional[np.ndarray] = dc_field(repr=False, default=None)
    scale: Optional[np.ndarray] = dc_field(repr=False, default=None)
    stencil: Optional[N.Handle] = dc_field(repr=False, default=None, compare=False)
    stencil_device: int = dc_field(repr=False, default=0, compare=False)

    def __len__(self) -> int:
        return len(self.target_global)

    def export_rows(self) -> List[dict]:
        return [
            {
                "target_global_index": int(self.target_global[k]),
                "source_global_indices": [int(self.source_global[n]) for n in self.nodes[k]],
                "weights": [float(w) for w in self.weights[k]],
                "fallback": bool(self.fallback[k]),
            }
            for k in range(len(self))
        ]

    def device_stencil(self, device: int) -> int:
        """Device stencil handle on ``device`` (uploaded from the host arrays if the weights
        were built elsewhere or on another device)."""
        if self.stencil is None or self.stencil_device != device:
            nodes = np.ascontiguousarray(self.nodes, dtype=np.int64)
            w = np.ascontiguousarray(self.weights, dtype=np.float64)
            h = C.c_uint64(0)
            N.call("sg_stencil_create_k", device, N.ptr(nodes), N.ptr(w), len(self), nodes.shape[1],
                   self.source_nnodes, N.ref(h))
            self.stencil, self.stencil_device = N.Handle(h.value), device
        return self.stencil.handle

    def _staging(self, device: int, src_shape, dst_shape, nfields: int = 1):
        """Device staging pairs for host-resident fields, cached per (device, shapes, F)."""
        key = (device, tuple(src_shape), tuple(dst_shape), nfields)
        cache = self.__dict__.setdefault("_staging_cache", {})
        if key not in cache:
            cache.clear()
            cache[key] = ([DeviceArray(src_shape[0], src_shape[1], np.float64, device) for _ in range(nfields)],
                          [DeviceArray(dst_shape[0], dst_shape[1], np.float64, device) for _ in range(nfields)])
        return cache[key]

    def _scratch(self, device: int, shape, index: int) -> DeviceArray:
        """Device result buffer ``index`` of ``shape`` for apply_remap_fields, cached."""
        key = (device, tuple(shape), index)
        cache = self.__dict__.setdefault("_scratch_cache", {})
        if key not in cache:
            cache[key] = DeviceArray(shape[0], shape[1], np.float64, device)
        return cache[key]

    def distinct_sources(self) -> int:
        u = C.c_int64()
        N.call("sg_stencil_info", self.device_stencil(self.stencil_device), None, None, N.ref(u))
        return u.value


def build_remap(source_fs: NodeColumns, target: Grid, target_dist: Distribution, ctx=None,
                allow_fallback: bool = False, locator: Optional[MeshLocator] = None) -> InterpolationWeights:
    """Weights remapping source node fields onto this partition's owned target points
    (interp.py:154-203).  Zero communication."""
    mesh = source_fs.mesh
    owned = np.flatnonzero(target_dist.part_of == mesh.partition_id).astype(np.int64)
    pts = np.ascontiguousarray(target.xyz()[owned])
    loc = locator if locator is not None else MeshLocator(mesh)
    m = len(owned)
    nodes = np.zeros((m, 3), np.int64)
    weights = np.zeros((m, 3))
    scale = np.ones(m)
    fb = np.zeros(m, np.uint8)
    status = np.zeros(m, np.uint8)
    first_bad = C.c_int64(-1)
    h = C.c_uint64(0)
    rc = N.lib.sg_remap_build(loc.handle, N.ptr(pts), m, mesh.nb_nodes, int(bool(allow_fallback)), N.ref(h),
                              N.ptr(nodes), N.ptr(weights), N.ptr(scale), N.ptr(fb), N.ptr(status),
                              N.ref(first_bad))
    if rc != N.SG_OK:
        msg = N.last_error()
        if first_bad.value >= 0:
            t = int(owned[first_bad.value])
            if msg.startswith("NotLocated"):
                raise NotLocated(
                    f"target point {t} not located in local source elements; increase the source mesh halo depth",
                    target_global_index=t,
                )
            if "singular" in msg:
                raise DegenerateTriangle("singular vertex matrix")  # interp.py:66-67
            if "origin" in msg:
                raise DegenerateTriangle("projection plane through the origin")  # interp.py:69-70
            raise DegenerateTriangle(f"degenerate candidate triangle near target point {t}")
        N.check(rc)
    return InterpolationWeights(
        target_global=owned, nodes=nodes, weights=weights, fallback=fb.astype(bool),
        source_nnodes=mesh.nb_nodes, source_global=mesh.node_global, scale=scale,
        stencil=N.Handle(h.value), stencil_device=loc.device,
    )


def _check_shapes(weights: InterpolationWeights, src: Field, dst: Field) -> None:
    if src.npts != weights.source_nnodes:
        raise ShapeMismatch(f"source field has {src.npts} points, weights expect {weights.source_nnodes}")
    if dst.npts != len(weights):
        raise ShapeMismatch(f"target field has {dst.npts} points, weights cover {len(weights)}")
    if src.levels != dst.levels:
        raise ShapeMismatch("level counts differ")


def apply_remap_device(weights: InterpolationWeights, sources: Sequence[DeviceArray],
                       targets: Sequence[DeviceArray], variant: int = APPLY_DEFAULT, stream: int = 0) -> None:
    """The kernel entry point: F device field pairs sharing one stencil, asynchronous on
    ``stream``."""
    if len(sources) != len(targets) or not sources:
        raise ValueError("need matching, non-empty source/target lists")
    dev = sources[0].device
    sh = weights.device_stencil(dev)
    s = np.array([a.handle for a in sources], np.uint64)
    t = np.array([a.handle for a in targets], np.uint64)
    N.call("sg_remap_apply", sh, N.ptr(s), N.ptr(t), len(s), variant, stream)


def apply_remap_range(weights: InterpolationWeights, sources: Sequence[DeviceArray], targets: Sequence[DeviceArray],
                      t0: int, t1: int, variant: int = APPLY_DEFAULT, stream: int = 0) -> None:
    """apply_remap_device restricted to targets [t0, t1) (sg_remap_apply_range)."""
    dev = sources[0].device
    sh = weights.device_stencil(dev)
    s = np.array([a.handle for a in sources], np.uint64)
    t = np.array([a.handle for a in targets], np.uint64)
    N.call("sg_remap_apply_range", sh, N.ptr(s), N.ptr(t), len(s), t0, t1, variant, stream)


def apply_remap_list(weights: InterpolationWeights, sources: Sequence[DeviceArray], targets: Sequence[DeviceArray],
                     target_list: DeviceArray, variant: int = APPLY_DEFAULT, stream: int = 0) -> None:
    """apply_remap_device for the targets listed in a device int32 array (sg_remap_apply_list)."""
    dev = sources[0].device
    s = np.array([a.handle for a in sources], np.uint64)
    t = np.array([a.handle for a in targets], np.uint64)
    N.call("sg_remap_apply_list", weights.device_stencil(dev), N.ptr(s), N.ptr(t), len(s), target_list.ptr,
           target_list.shape[0], variant, stream)


def apply_remap_fused_list(weights: InterpolationWeights, plan, source: DeviceArray, target: DeviceArray,
                           target_list: DeviceArray, peer_info, stream: int = 0) -> None:
    """apply_remap_fused for the targets listed in a device int32 array."""
    dev = source.device
    peers = plan.peers
    ptrs = np.array([peer_info[p][0] for p in peers] or [0], np.uint64)
    pitch = np.array([peer_info[p][1] for p in peers] or [0], np.int64)
    N.call("sg_remap_apply_fused_list", weights.device_stencil(dev), plan.native(dev), source.handle, target.handle,
           target_list.ptr, target_list.shape[0], N.ptr(ptrs), N.ptr(pitch), stream)


def apply_remap_fused(weights: InterpolationWeights, plan, source: DeviceArray, target: DeviceArray, t0: int,
                      t1: int, peer_info, stream: int = 0) -> None:
    """Targets [t0, t1) with ghost stencil rows read straight from their owners' fields
    (sg_remap_apply_fused): halo exchange + apply in one kernel.  peer_info[r] = (ptr,
    pitch, device) of rank r's source field (ctx.peer_fields); owners' rows must be final."""
    dev = source.device
    peers = plan.peers
    ptrs = np.array([peer_info[p][0] for p in peers] or [0], np.uint64)
    pitch = np.array([peer_info[p][1] for p in peers] or [0], np.int64)
    N.call("sg_remap_apply_fused", weights.device_stencil(dev), plan.native(dev), source.handle, target.handle,
           t0, t1, N.ptr(ptrs), N.ptr(pitch), stream)


def _auto_mode(weights: InterpolationWeights, mapped: bool) -> str:
    """Host-execute path chooser.  Moving only the referenced rows pays when the stencil skips
    a good share of the source rows (cfg5 bilinear reads every row -> dma).  Page-locked,
    mapped sources take the GPU gather, which needs no host CPU and was fastest on every box
    measured (profiles/r01_e2e_modes.md: 116 ms vs compact 124-143 ms vs dma 134-136 ms at cfg3).
    Pageable sources choose between host packing (compact) and plain DMA by timing the first
    calls, because host memory bandwidth decides it and differs between hosts."""
    n = max(weights.source_nnodes, 1)
    if weights.distinct_sources() >= 0.85 * n:
        return "dma"
    if mapped:
        return "gather"
    modes = ("compact", "dma")
    seen = weights.__dict__.setdefault("_auto_s", {})
    for m in modes:
        if len(seen.get(m, [])) < 2:  # the first call of a mode also builds its plan
            return m
    return min(modes, key=lambda m: min(seen[m]))


def _is_pinned(a: np.ndarray) -> bool:
    """True when ``a`` is page-locked by the library (PinnedArray, or registered by
    device.ensure_pinned)."""
    from .device import is_pinned

    return is_pinned(a)


def execute_host(weights: InterpolationWeights, host_src: Sequence[np.ndarray], host_dst: Sequence[np.ndarray],
                 dev_src: Sequence[DeviceArray], dev_dst: Sequence[DeviceArray], nchunks: int = 0,
                 variant: int = APPLY_DEFAULT, mode: str = "auto", direct_period: int = -1) -> int:
    """Host buffers in, host buffers out (sg_remap_execute_host): chunked h2d of the referenced
    source rows, apply, d2h of the target rows, overlapped on three streams.  Host arrays
    should be pinned (``device.PinnedArray``) for full PCIe rate.  mode: "dma" (chunked
    copies of the referenced row runs), "compact" (only referenced rows, packed on the host by
    the library's thread pool), "gather" (only referenced rows, read by a GPU kernel straight
    from the pinned, mapped source arrays into a compact device copy), "zerocopy" (the apply
    kernel reads/writes the pinned host arrays directly over PCIe), "auto" (times the
    candidates on the first calls and keeps the fastest; dma when the stencil reads >= 85 %
    of the source rows).
    Returns source rows moved."""
    dev = dev_src[0].device
    sh = weights.device_stencil(dev)
    m = len(weights)
    if nchunks <= 0:
        nchunks = int(max(1, min(64, m // 16384)))
    for a, d in zip(list(host_src) + list(host_dst), list(dev_src) + list(dev_dst)):
        if a.shape != d.shape or a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise ValueError("host arrays must be C-contiguous float64 of the device arrays' shape")
    hs = np.array([a.ctypes.data for a in host_src], np.uint64)
    hd = np.array([a.ctypes.data for a in host_dst], np.uint64)
    s = np.array([a.handle for a in dev_src], np.uint64)
    t = np.array([a.handle for a in dev_dst], np.uint64)
    rows = C.c_int64(0)
    tuned = mode == "auto"
    if tuned:
        mode = _auto_mode(weights, all(_is_pinned(a) for a in host_src))
    flags = {"dma": 0, "compact": 1, "zerocopy": 2, "gather": 4, "gather_warp": 4 | 8}[mode]
    if direct_period < 0:
        direct_period = HOST_EXECUTE_DIRECT_PERIOD
    if mode == "compact" and direct_period > 0:
        flags |= (min(int(direct_period), 255) << 8)  # every n-th chunk: one direct DMA
    t0 = time.perf_counter()
    N.call("sg_remap_execute_host", sh, N.ptr(s), N.ptr(t), len(s), N.ptr(hs), N.ptr(hd), nchunks, variant,
           flags, N.ref(rows))
    if tuned:
        weights.__dict__.setdefault("_auto_s", {}).setdefault(mode, []).append(time.perf_counter() - t0)
    return rows.value


def apply_remap(weights: InterpolationWeights, source_field: Field, target_field: Field) -> None:
    """target[t] = sum_i w_i * source[node_i], every level (interp.py:206-228).

    The reference's contract, whatever mirrors the fields have: the result lands in
    ``target_field.host`` and the target goes SYNCED -> HOST_DIRTY (HOST_ONLY and the
    reference's DEVICE_DIRTY quirk stay as they are).  The arithmetic always runs on the
    GPU; see ``apply_remap_fields``.  ``apply_remap_device_fields`` is the HBM-only entry
    point (target left DEVICE_DIRTY)."""
    apply_remap_fields(weights, [source_field], [target_field])


def _device_current(f: Field, dev: int) -> bool:
    return f.device is not None and f.device.device == dev and f.kind.dtype == np.float64


def apply_remap_device_fields(weights: InterpolationWeights, source_fields: Sequence[Field],
                              target_fields: Sequence[Field], stream: int = 0) -> None:
    """The HBM-only apply (SURVEY.md §8(b) device entry point): F float64 field pairs whose
    device mirrors are current (SYNCED or DEVICE_DIRTY), one kernel launch, targets left
    DEVICE_DIRTY.  No host copy; ``update_host`` brings the result down."""
    if len(source_fields) != len(target_fields) or not source_fields:
        raise ValueError("need matching, non-empty source/target field lists")
    dev = current_device()
    for s, t in zip(source_fields, target_fields):
        _check_shapes(weights, s, t)
        for f in (s, t):
            if f.state is MemoryState.HOST_ONLY or f.device is None:
                raise NoDevice(f"field {f.name!r} has no device buffer")
            if f.state is MemoryState.HOST_DIRTY:
                raise StaleDevice(f"device access to {f.name!r} while host is newer; update_device first")
            if not _device_current(f, dev):
                raise ValueError(f"field {f.name!r}: device apply needs float64 mirrors on device {dev}")
    apply_remap_device(weights, [s.device for s in source_fields], [t.device for t in target_fields], stream=stream)
    N.call("sg_stream_synchronize", dev, stream)
    for t in target_fields:
        t.mark_device_written()


def apply_remap_fields(weights: InterpolationWeights, source_fields: Sequence[Field],
                       target_fields: Sequence[Field]) -> None:
    """apply_remap for F field pairs sharing one stencil, with the reference's contract
    (interp.py:218-228: reads ``source.host``, writes ``target.host``, SYNCED -> HOST_DIRTY).

    * Sources whose device mirror is bit-identical to the host (SYNCED) are read from HBM:
      one kernel launch for all such pairs, written into the target's device buffer when
      that buffer's contents are not observable (target SYNCED or HOST_DIRTY) or into a
      staging buffer otherwise, then one d2h of the target rows into ``target.host``.
    * Every other source (HOST_ONLY, HOST_DIRTY, and DEVICE_DIRTY, whose host copy is what
      the reference reads) goes through the pipelined host-buffer execute."""
    if len(source_fields) != len(target_fields) or not source_fields:
        raise ValueError("need matching, non-empty source/target field lists")
    for s, t in zip(source_fields, target_fields):
        _check_shapes(weights, s, t)
    dev = current_device()

    pairs = list(zip(source_fields, target_fields))
    on_dev = [p for p in pairs if p[0].state is MemoryState.SYNCED and _device_current(p[0], dev)]
    on_host = [p for p in pairs if not (p[0].state is MemoryState.SYNCED and _device_current(p[0], dev))]
    if on_dev:
        outs = []
        for k, (_, t) in enumerate(on_dev):
            if _device_current(t, dev) and t.state in (MemoryState.SYNCED, MemoryState.HOST_DIRTY):
                outs.append(t.device)
            else:
                outs.append(weights._scratch(dev, t.shape, k))
        apply_remap_device(weights, [s.device for s, _ in on_dev], outs)
        for (_, t), o in zip(on_dev, outs):
            th = t.host
            if th.dtype == np.float64 and th.flags["C_CONTIGUOUS"] and th.flags["WRITEABLE"]:
                o.download(th)
            else:
                th[:] = o.to_numpy()
            if t.state is MemoryState.SYNCED:
                t.state = MemoryState.HOST_DIRTY
    if not on_host:
        return
    # host-resident fields: reference semantics (reads source.host, writes target.host);
    # the arithmetic runs on the device through staging buffers cached on the weights
    shapes = {(s.shape, t.shape) for s, t in on_host}
    groups = [on_host] if len(shapes) == 1 else [[p] for p in on_host]
    for group in groups:
        srcs, dsts = weights._staging(dev, group[0][0].shape, group[0][1].shape, len(group))
        host_src, outs, copy_back = [], [], []
        for s, t in group:
            h = s.host
            if h.dtype != np.float64 or not h.flags["C_CONTIGUOUS"]:
                h = np.ascontiguousarray(h, dtype=np.float64)
            host_src.append(h)
            th = t.host
            direct = th.dtype == np.float64 and th.flags["C_CONTIGUOUS"] and th.flags["WRITEABLE"]
            out = th if direct else np.empty(t.shape, np.float64)
            outs.append(out)
            copy_back.append(None if direct else (th, out))
        from .device import ensure_pinned

        for s, t in group:  # the fields' own large numpy arrays: page-locked once, for their lifetime
            ensure_pinned(s.host)
            ensure_pinned(t.host)
        moved = execute_host(weights, host_src, outs, srcs, dsts, nchunks=HOST_EXECUTE_CHUNKS,
                             mode=HOST_EXECUTE_MODE)
        weights.__dict__["last_host_rows_moved"] = moved  # source rows per field that crossed PCIe
        for cb in copy_back:
            if cb is not None:
                cb[0][:] = cb[1]
        for _, t in group:
            if t.state is MemoryState.SYNCED:
                t.state = MemoryState.HOST_DIRTY


def export_weights(weights: InterpolationWeights, stream) -> None:
    import json

    for row in weights.export_rows():
        stream.write(json.dumps(row) + "\n")


def build_bilinear(source_fs: NodeColumns, target: Grid, target_dist: Distribution, ctx=None
                   ) -> InterpolationWeights:
    """Structured-bilinear weights (4 nodes per target) onto this partition's owned target
    points — BASELINE configs[4].  The reference has no such method; the definition is in
    csrc/bilinear.cu and oracle/oracle.py:bilinear_stencil (parity unpinned vs the
    reference).  Zero communication; NotLocated if a bracketing node is outside the local
    (owned + halo) mesh."""
    mesh = source_fs.mesh
    grid = mesh.grid
    owned = np.flatnonzero(target_dist.part_of == mesh.partition_id).astype(np.int64)
    ll = np.ascontiguousarray(target.lonlats()[owned])
    m = len(owned)
    nodes = np.zeros((m, 4), np.int64)
    weights = np.zeros((m, 4))
    status = np.zeros(m, np.uint8)
    lat = np.ascontiguousarray(grid.latitudes, dtype=np.float64)
    nl = np.ascontiguousarray(grid.nlons, dtype=np.int64)
    ng = np.ascontiguousarray(mesh.node_global, dtype=np.int64)
    h = C.c_uint64(0)
    bad = C.c_int64(-1)
    dev = current_device()
    rc = N.lib.sg_bilinear_build(dev, grid.nrows, N.ptr(lat), N.ptr(nl), int(mesh.include_pole), N.ptr(ng),
                                 mesh.nb_nodes, N.ptr(ll), m, N.ref(h), N.ptr(nodes), N.ptr(weights),
                                 N.ptr(status), N.ref(bad))
    if rc != N.SG_OK:
        msg = N.last_error()
        if bad.value >= 0:
            t = int(owned[bad.value])
            raise NotLocated(f"target point {t} not located in local source elements; increase the source mesh "
                             "halo depth", target_global_index=t)
        N.check(rc)
    return InterpolationWeights(
        target_global=owned, nodes=nodes, weights=weights, fallback=np.zeros(m, bool),
        source_nnodes=mesh.nb_nodes, source_global=mesh.node_global, scale=np.ones(m),
        stencil=N.Handle(h.value), stencil_device=dev,
    )


class Interpolation:
    """Atlas-style operator: ``Interpolation(source_fs, target, target_dist, ctx).execute(src,
    tgt)`` builds the stencil once and applies it per call.  ``method``:
    "finite-element" (the reference's gnomonic triangles) or "structured-bilinear"."""

    def __init__(self, source_fs: NodeColumns, target: Grid, target_dist: Distribution, ctx=None,
                 allow_fallback: bool = False, method: str = "finite-element"):
        if method == "finite-element":
            self.weights = build_remap(source_fs, target, target_dist, ctx, allow_fallback)
        elif method == "structured-bilinear":
            self.weights = build_bilinear(source_fs, target, target_dist, ctx)
        else:
            raise ValueError(f"unknown interpolation method {method!r}")

    def execute(self, source_field: Field, target_field: Field) -> None:
        apply_remap(self.weights, source_field, target_field)

    def execute_device(self, source_field: Field, target_field: Field) -> None:
        """HBM-only execute: device-current mirrors in, target left DEVICE_DIRTY."""
        apply_remap_device_fields(self.weights, [source_field], [target_field])
