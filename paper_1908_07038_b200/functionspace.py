"""Function spaces and the halo exchange (functionspace.py:1-258 of the reference).

``NodeColumns`` binds fields to one partition's mesh nodes; its constructor builds the
exchange plan with the reference's protocol (one request message per other rank, tag 101,
functionspace.py:58-94).  The exchange itself runs on the GPU:

* ``halo_exchange(plan, f, ctx)`` — the reference entry point with the reference semantics
  (PlanMismatch, StaleHost on DEVICE_DIRTY, SYNCED -> HOST_DIRTY, one counted message per
  peer with the payload's byte length, functionspace.py:107-118).  The ghost values are
  moved by device kernels: through the field's own device mirror when it is current
  (SYNCED), otherwise through a device staging copy of the host rows; the received ghost
  rows are copied back into ``f.host``.
* ``halo_exchange_device(plan, f, ctx)`` — device-resident fields (SYNCED / DEVICE_DIRTY):
  exchange in HBM only, field left DEVICE_DIRTY (SURVEY.md §8(b) "device entry points").

Transport: ranks of one process (``run_ranks``) use one fused pull kernel over peer memory;
one process per GPU (``DistContext``) uses pack -> grouped NCCL send/recv -> unpack.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field
from typing import Dict, Optional

import numpy as np

from . import _native as N
from .device import DeviceArray, current_device
from .errors import InconsistentMesh, PlanMismatch, StaleHost
from .field import Field, Kind, MemoryState, _host_mirror, create_field
from .grid import Grid
from .mesh import Mesh
from .partition import Distribution

_TAG_PLAN_REQUEST = 101  # functionspace.py:24
_TAG_EXCHANGE = 102  # functionspace.py:25


def row_runs(rows: np.ndarray) -> np.ndarray:
    """(row0, nrows) runs, ascending and maximal, covering the distinct values of ``rows``."""
    rows = np.unique(np.asarray(rows, np.int64))
    if len(rows) == 0:
        return np.empty((0, 2), np.int64)
    cut = np.flatnonzero(np.diff(rows) != 1) + 1
    starts = rows[np.concatenate([[0], cut])]
    ends = rows[np.concatenate([cut - 1, [len(rows) - 1]])] + 1
    return np.stack([starts, ends - starts], axis=1).astype(np.int64)


@dataclass
class HaloExchangePlan:
    """Per peer: owned local rows to send (requester's order) and ghost local rows to
    receive ((halo, gidx) order); ``recv_remote`` adds each ghost's row on its owner
    (mesh.py:303-308), which is what the peer-memory pull kernel reads."""

    nnodes: int
    send: Dict[int, np.ndarray] = dc_field(default_factory=dict)
    recv: Dict[int, np.ndarray] = dc_field(default_factory=dict)
    recv_remote: Dict[int, np.ndarray] = dc_field(default_factory=dict)
    _native: Dict[int, N.Handle] = dc_field(default_factory=dict, repr=False)
    _send_runs: Optional[np.ndarray] = dc_field(default=None, repr=False)

    def send_runs(self) -> np.ndarray:
        """(row0, nrows) runs covering the union of the send lists, ascending."""
        if self._send_runs is None:
            self._send_runs = row_runs(np.concatenate([np.asarray(v, np.int64) for v in self.send.values()])
                                       if self.send else np.empty(0, np.int64))
        return self._send_runs

    @property
    def peers(self):
        return sorted(set(self.send) | set(self.recv))

    @property
    def ghost_rows(self) -> Optional[tuple]:
        """[lo, hi) spanning every received row (ghosts are numbered last)."""
        if not self.recv:
            return None
        allr = np.concatenate(list(self.recv.values()))
        return int(allr.min()), int(allr.max()) + 1

    def native(self, device: int) -> int:
        h = self._native.get(device)
        if h is None:
            peers = self.peers
            arr = lambda d, p: d.get(p, np.empty(0, np.int64))  # noqa: E731
            sc = np.array([len(arr(self.send, p)) for p in peers], np.int64)
            rc = np.array([len(arr(self.recv, p)) for p in peers], np.int64)
            cat = lambda parts: np.ascontiguousarray(  # noqa: E731
                np.concatenate(parts) if parts else np.empty(0), dtype=np.int64)
            srows = cat([arr(self.send, p) for p in peers])
            rrows = cat([arr(self.recv, p) for p in peers])
            rrem = cat([arr(self.recv_remote, p) if p in self.recv_remote else
                        np.full(len(arr(self.recv, p)), -1) for p in peers])
            pv = np.array(peers, np.int32)
            out = C.c_uint64(0)
            N.call("sg_halo_plan_create", device, self.nnodes, len(peers), N.ptr(pv), N.ptr(sc), N.ptr(srows),
                   N.ptr(rc), N.ptr(rrows), N.ptr(rrem), N.ref(out))
            h = self._native[device] = N.Handle(out.value)
        return h.handle

    # -- device transports --------------------------------------------------------------------
    def complete_remote(self, me: int, peer_sends) -> None:
        """Fill ``recv_remote`` for peers it lacks (a plan built from send/recv lists only)
        from the owners' send lists: ``peer_sends[p]`` = rank p's ``send`` dict, whose entry
        for this rank lists, in this rank's receive order, the owner rows of our ghosts
        (functionspace.py:83-93).  The pull/fused kernels need them; the library refuses a
        plan without them rather than read a wrong row."""
        missing = [p for p in self.recv if p not in self.recv_remote]
        if not missing:
            return
        for p in missing:
            rows = peer_sends[p].get(me)
            if rows is None or len(rows) != len(self.recv[p]):
                raise PlanMismatch(f"rank {p} sends {0 if rows is None else len(rows)} rows, "
                                   f"this rank expects {len(self.recv[p])}")
            self.recv_remote[p] = np.asarray(rows, np.int64)
        for h in self._native.values():
            h.close()
        self._native.clear()

    def pull(self, dev: DeviceArray, peer_info, stream: int = 0) -> None:
        """peer_info[r] = (ptr, pitch, device) of rank r's field; one fused kernel on
        ``stream``."""
        peers = self.peers
        ptrs = np.array([peer_info[p][0] for p in peers] or [0], np.uint64)
        pitch = np.array([peer_info[p][1] for p in peers] or [0], np.int64)
        N.call("sg_halo_pull", self.native(dev.device), dev.handle, N.ptr(ptrs), N.ptr(pitch), stream)

    def exchange_nccl(self, dev: DeviceArray, comm: int, stream: int = 0) -> None:
        N.call("sg_halo_exchange_nccl", self.native(dev.device), dev.handle, comm, stream)

    def pack(self, dev: DeviceArray, sendbuf_ptr: int, stream: int = 0) -> None:
        N.call("sg_halo_pack", self.native(dev.device), dev.handle, sendbuf_ptr, stream)

    def unpack(self, dev: DeviceArray, recvbuf_ptr: int, stream: int = 0) -> None:
        N.call("sg_halo_unpack", self.native(dev.device), dev.handle, recvbuf_ptr, stream)


def build_exchange_plan(mesh: Mesh, ctx) -> HaloExchangePlan:
    """Request/response plan build (functionspace.py:58-94): every rank sends each other
    rank the global ids it needs from it (possibly none); owners answer by mapping them to
    owned local rows in the requested order."""
    plan = HaloExchangePlan(nnodes=mesh.nb_nodes)
    if ctx is None or ctx.nranks == 1:
        return plan
    ghosts = np.flatnonzero(mesh.node_ghost)
    owner = mesh.node_part[ghosts]
    for p in np.unique(owner):
        rows = ghosts[owner == p]
        plan.recv[int(p)] = rows
        plan.recv_remote[int(p)] = mesh.node_remote[rows].astype(np.int64)
    owned_gid = mesh.node_global[~mesh.node_ghost]
    # owned local rows are 0..n_owned-1 in ascending gid: a sorted lookup replaces the dict
    for peer in range(ctx.nranks):
        if peer != ctx.rank:
            want = plan.recv.get(peer)
            gids = mesh.node_global[want] if want is not None else np.empty(0, np.int64)
            ctx.send(peer, _TAG_PLAN_REQUEST, np.asarray(gids, np.int64).tobytes())
    for peer in range(ctx.nranks):
        if peer == ctx.rank:
            continue
        req = np.frombuffer(ctx.receive(peer, _TAG_PLAN_REQUEST), dtype=np.int64)
        if len(req) == 0:
            continue
        pos = np.searchsorted(owned_gid, req)
        bad = (pos >= len(owned_gid)) | (owned_gid[np.minimum(pos, len(owned_gid) - 1)] != req)
        if np.any(bad):
            g = int(req[np.argmax(bad)])
            raise InconsistentMesh(f"rank {ctx.rank} asked for global index {g} it does not own")
        plan.send[peer] = pos.astype(np.int64)
    return plan


def _count_messages(plan: HaloExchangePlan, f: Field, ctx) -> None:
    """The reference sends one message per send-peer and receives one per recv-peer
    (functionspace.py:113-117); keep the counters identical."""
    row_bytes = f.levels * f.host.dtype.itemsize
    for peer in sorted(plan.send):
        ctx.messages_sent += 1
        ctx.bytes_sent += len(plan.send[peer]) * row_bytes
    ctx.messages_received += len(plan.recv)


def _staging(f: Field) -> DeviceArray:
    st = getattr(f, "_halo_staging", None)
    dev = current_device()
    if st is None or st.device != dev:
        st = DeviceArray(f.npts, f.levels, f.kind.dtype, dev)
        object.__setattr__(f, "_halo_staging", st)
    return st


def halo_exchange(plan: HaloExchangePlan, f: Field, ctx) -> None:
    """Copy owner values into every ghost row, all levels (functionspace.py:107-118)."""
    if f.npts != plan.nnodes:
        raise PlanMismatch(f"field has {f.npts} points, plan covers {plan.nnodes} nodes")
    if f.state is MemoryState.DEVICE_DIRTY:
        raise StaleHost(f"field {f.name!r} is device-dirty; update_host before exchanging")
    if ctx is not None and getattr(ctx, "nranks", 1) > 1:
        if f.state is MemoryState.SYNCED and f.device is not None and f.device.device == current_device():
            dev = f.device
        else:  # stage only the rows peers read (the union of the send lists), not the field
            dev = _staging(f)
            h = f.host
            from .device import ensure_pinned

            runs = plan.send_runs()
            # page-locked mirrors (large ones are pinned here): one pull kernel reads the runs
            # straight from host memory; few runs: one DMA each; many runs from a small pageable
            # array: one DMA of the whole field beats a staged copy per run
            if h.dtype == dev.dtype and h.flags["C_CONTIGUOUS"] and (ensure_pinned(h) or len(runs) <= 16):
                dev.upload_row_runs(h, runs)
            else:
                dev.upload(h)
        ctx.device_exchange(plan, dev)
        span = plan.ghost_rows
        if span is not None:
            lo, hi = span
            out = f.host[lo:hi]
            if out.dtype == dev.dtype and out.flags["C_CONTIGUOUS"]:
                dev.download_rows_into(lo, out)  # straight into the (page-locked) mirror
            else:
                out[...] = dev.download_rows(lo, hi - lo)
        _count_messages(plan, f, ctx)
    if f.state is MemoryState.SYNCED:
        f.state = MemoryState.HOST_DIRTY


def halo_exchange_device(plan: HaloExchangePlan, f: Field, ctx) -> None:
    """Device-resident exchange: field must be SYNCED or DEVICE_DIRTY; ends DEVICE_DIRTY."""
    if f.npts != plan.nnodes:
        raise PlanMismatch(f"field has {f.npts} points, plan covers {plan.nnodes} nodes")
    if f.state in (MemoryState.HOST_ONLY, MemoryState.HOST_DIRTY):
        from .errors import StaleDevice

        raise StaleDevice(f"field {f.name!r} has no current device mirror; update_device first")
    if ctx is not None and getattr(ctx, "nranks", 1) > 1:
        ctx.device_exchange(plan, f.device)
        _count_messages(plan, f, ctx)
    f.mark_device_written()


class NodeColumns:
    """Fields on the nodes (owned + ghost) of one partition's mesh (functionspace.py:121-154)."""

    def __init__(self, mesh: Mesh, ctx=None):
        self.mesh = mesh
        self.halo = mesh.halo_depth
        self.exchange_plan = build_exchange_plan(mesh, ctx)
        self._owned = ~mesh.node_ghost

    @property
    def nb_nodes(self) -> int:
        return self.mesh.nb_nodes

    @property
    def owned_global(self) -> np.ndarray:
        return self.mesh.node_global[self._owned]

    @property
    def global_size(self) -> int:
        return self.mesh.grid.npts + (2 if self.mesh.include_pole else 0)

    def owned_rows(self, f: Field) -> np.ndarray:
        return f.host[self._owned]

    def owned_row_index(self) -> np.ndarray:
        return np.flatnonzero(self._owned)

    def create_field(self, name: str, levels: int = 1, kind: Kind = Kind.REAL64) -> Field:
        f = create_field(name, (self.mesh.nb_nodes, levels), kind)
        f.functionspace_tag = f"nodes:{self.mesh.grid.name}:p{self.mesh.partition_id}"
        return f

    def halo_exchange(self, f: Field, ctx=None) -> None:
        halo_exchange(self.exchange_plan, f, ctx)

    def halo_exchange_device(self, f: Field, ctx=None) -> None:
        halo_exchange_device(self.exchange_plan, f, ctx)


class StructuredColumns:
    """Fields on the owned points of a distributed grid; rows = owned gids ascending, the
    row order of InterpolationWeights.target_global (functionspace.py:157-182)."""

    def __init__(self, grid: Grid, dist: Distribution, part: int = 0):
        self.grid = grid
        self.dist = dist
        self.part = part
        self.local_points = np.flatnonzero(dist.part_of == part).astype(np.int64)

    @property
    def owned_global(self) -> np.ndarray:
        return self.local_points

    @property
    def global_size(self) -> int:
        return self.grid.npts

    def owned_rows(self, f: Field) -> np.ndarray:
        return f.host

    def owned_row_index(self) -> np.ndarray:
        return np.arange(len(self.local_points))

    def create_field(self, name: str, levels: int = 1, kind: Kind = Kind.REAL64) -> Field:
        f = create_field(name, (len(self.local_points), levels), kind)
        f.functionspace_tag = f"structured:{self.grid.name}:p{self.part}"
        return f


# -- output / verification plumbing (functionspace.py:185-258) ---------------------------------
_TAG_SCATTER = 104  # functionspace.py:27


def _owned_device_rows(fs, f: Field):
    """(DeviceArray, row0, nrows) holding the current owned values of ``f``: the field's own
    mirror when it is current and the owned rows are contiguous, else a staging upload."""
    rows = fs.owned_row_index()
    contiguous = len(rows) == 0 or (rows[0] == 0 and rows[-1] == len(rows) - 1)
    if f.device is not None and f.state in (MemoryState.SYNCED, MemoryState.DEVICE_DIRTY) and contiguous:
        return f.device, 0, len(rows)
    if f.state is MemoryState.DEVICE_DIRTY:
        f.update_host()
    # owned rows [0, n): upload straight from the host mirror (page-locked for large fields)
    host = f.host[:len(rows)] if contiguous and f.host.flags["C_CONTIGUOUS"] else np.ascontiguousarray(f.host[rows])
    st = DeviceArray(max(len(rows), 1), f.levels, f.host.dtype, current_device())
    if len(rows):
        st.upload_rows(0, host)
    return st, 0, len(rows)


def checksum(fs, f: Field, ctx) -> int:
    """Partition-invariant 64-bit digest of the owned values (functionspace.py:233-254),
    computed by a device kernel (sg_field_checksum); ranks combine partials exactly like the
    reference (gather_to_root + broadcast_from_root).  A DEVICE_DIRTY field is digested from
    its (current) device mirror."""
    dev, row0, n = _owned_device_rows(fs, f)
    gids = np.ascontiguousarray(fs.owned_global, dtype=np.int64)
    part = C.c_uint64(0)
    N.call("sg_field_checksum", dev.handle, row0, n, N.ptr(gids), N.ref(part))
    partial = np.uint64(part.value)
    if ctx is None or ctx.nranks == 1:
        return int(partial)
    parts = ctx.gather_to_root(partial.tobytes())
    digest = None
    if ctx.rank == 0:
        total = np.uint64(0)
        with np.errstate(over="ignore"):
            for blob in parts:
                total += np.frombuffer(blob, dtype=np.uint64)[0]
        digest = total.tobytes()
    return int(np.frombuffer(ctx.broadcast_from_root(digest), dtype=np.uint64)[0])


def format_checksum(digest: int) -> str:
    return f"{digest:016x}"


def _owned_values(fs, f: Field) -> np.ndarray:
    if f.state is MemoryState.DEVICE_DIRTY:
        rows = fs.owned_row_index()
        if len(rows) and rows[0] == 0 and rows[-1] == len(rows) - 1:
            return f.device.download_rows(0, len(rows))
        f.update_host()
    return fs.owned_rows(f)


def _gids_device(gids: np.ndarray, device: int) -> DeviceArray:
    d = DeviceArray(max(len(gids), 1), 1, np.int64, device)
    if len(gids):
        d.upload(np.ascontiguousarray(gids, np.int64).reshape(-1, 1))
    return d


def _rows_copy(device: int, dst: DeviceArray, dst_idx: Optional[DeviceArray], src_ptr: int, src_pitch_bytes: int,
               src_idx: Optional[DeviceArray], n: int, row_bytes: int, stream: int = 0) -> None:
    N.call("sg_rows_copy", device, dst.ptr, dst.pitch * dst.dtype.itemsize, dst_idx.ptr if dst_idx is not None else 0,
           src_ptr, src_pitch_bytes, src_idx.ptr if src_idx is not None else 0, n, row_bytes, stream)


def _device_path(fs) -> bool:
    # every owned-row layout here is rows [0, n_owned): NodeColumns numbers owned nodes first,
    # StructuredColumns rows are all owned
    rows = fs.owned_row_index()
    return len(rows) == 0 or (rows[0] == 0 and rows[-1] == len(rows) - 1)


def gather_field(fs, f: Field, ctx) -> Optional[np.ndarray]:
    """Owned values of every rank assembled on rank 0 in global order (functionspace.py:185-204),
    on the device: rank 0 copies every rank's owned rows straight out of that rank's HBM
    (NVLink P2P / CUDA IPC) into their global rows of one device array (sg_rows_copy), then one
    D2H.  Device-current fields are read from their mirror, host ones through one staging
    upload.  Message counters as the reference: every other rank sends rank 0 one message of
    its gids and values."""
    single = ctx is None or ctx.nranks == 1
    device_path = _device_path(fs)
    if not single:  # collective decision: every rank takes the same path
        device_path = all(ctx.share(bool(device_path)))
    if not device_path:
        return _gather_host(fs, f, ctx)
    dev, _, n = _owned_device_rows(fs, f)
    L, dt = f.levels, f.host.dtype
    row_bytes = L * dt.itemsize
    gids = np.ascontiguousarray(fs.owned_global, np.int64)
    device = dev.device
    peers = None if single else ctx.peer_fields(dev)  # collective: every rank's owned rows
    if not single:
        parts = ctx.gather_to_root(gids.tobytes())  # the reference's message: gids + values
        if ctx.rank != 0:
            ctx.bytes_sent += n * row_bytes
            ctx.barrier()  # rank 0 has read my rows
            return None
    out = _host_mirror((fs.global_size, L), dt)  # page-locked when large: D2H at the DMA rate
    G = DeviceArray(max(fs.global_size, 1), L, dt, device)  # zero-filled, like np.zeros
    try:
        srcs = [(gids, dev.ptr, dev.pitch * dt.itemsize)] if single else [
            (np.frombuffer(parts[r], np.int64), peers[r][0], peers[r][1] * dt.itemsize) for r in range(ctx.nranks)]
        for g, ptr, pitch in srcs:
            if len(g):
                gd = _gids_device(g, device)
                _rows_copy(device, G, gd, ptr, pitch, None, len(g), row_bytes)
                gd.close()
        if fs.global_size:
            G.download(out)
    finally:
        if not single:
            ctx.barrier()
        G.close()
    return out


def _gather_host(fs, f: Field, ctx) -> Optional[np.ndarray]:
    owned = np.ascontiguousarray(_owned_values(fs, f))
    gids = fs.owned_global
    if ctx is None or ctx.nranks == 1:
        out = np.zeros((fs.global_size, f.levels), dtype=f.host.dtype)
        out[gids] = owned
        return out
    parts = ctx.gather_to_root(np.asarray(gids, np.int64).tobytes() + owned.tobytes())
    if ctx.rank != 0:
        return None
    out = np.zeros((fs.global_size, f.levels), dtype=f.host.dtype)
    row = 8 + f.host.dtype.itemsize * f.levels
    for blob in parts:
        n = len(blob) // row
        g = np.frombuffer(blob[: 8 * n], dtype=np.int64)
        out[g] = np.frombuffer(blob[8 * n:], dtype=f.host.dtype).reshape(n, f.levels)
    return out


def scatter_field(fs, f: Field, ctx, global_values: Optional[np.ndarray]) -> None:
    """Rank 0's global array into every rank's owned rows (functionspace.py:207-224), on the
    device: rank 0 uploads the global array once; every rank pulls its owned rows from rank
    0's HBM by global index (sg_rows_copy over P2P / CUDA IPC) and downloads them into its
    host rows.  Host rows written, SYNCED -> HOST_DIRTY, message counters as the reference
    (gid lists to rank 0, one data message back to every rank)."""
    if f.state is MemoryState.DEVICE_DIRTY:
        raise StaleHost(f"field {f.name!r} is device-dirty; update_host before scattering")
    single = ctx is None or ctx.nranks == 1
    root = single or ctx.rank == 0
    dt, L = f.host.dtype, f.levels
    same_dtype = not root or (isinstance(global_values, np.ndarray) and global_values.dtype == dt
                              and global_values.shape == (fs.global_size, L))
    device_path = _device_path(fs) and same_dtype
    if not single:  # collective decision (the reference's byte-reinterpreting quirk stays on the host)
        device_path = all(ctx.share(bool(device_path)))
    if not device_path:
        return _scatter_host(fs, f, ctx, global_values)
    rows = fs.owned_row_index()
    n = len(rows)
    gids = np.ascontiguousarray(fs.owned_global, np.int64)
    row_bytes = L * dt.itemsize
    device = current_device()
    G = None
    if root:
        G = DeviceArray(max(fs.global_size, 1), L, dt, device)
        if fs.global_size:
            G.upload(np.ascontiguousarray(global_values))
    mine = DeviceArray(max(n, 1), L, dt, device)
    try:
        if single:
            src = (G.ptr, G.pitch)
        else:
            src = ctx.peer_fields(G if root else mine)[0][:2]  # collective: rank 0's global copy
            counts = ctx.share(n)
            if root:
                ctx.messages_received += ctx.nranks - 1
                ctx.messages_sent += ctx.nranks - 1
                ctx.bytes_sent += sum(counts[1:]) * row_bytes
            else:
                ctx.messages_sent += 1
                ctx.bytes_sent += 8 * n
                ctx.messages_received += 1
        if n:
            gd = _gids_device(gids, device)
            _rows_copy(device, mine, None, src[0], src[1] * dt.itemsize, gd, n, row_bytes)
            mine.download_rows_into(0, f.host[:n])  # owned rows are [0, n)
            gd.close()
    finally:
        if not single:
            ctx.barrier()  # rank 0's global copy is no longer read
        mine.close()
        if G is not None:
            G.close()
    if f.state is MemoryState.SYNCED:
        f.state = MemoryState.HOST_DIRTY


def _scatter_host(fs, f: Field, ctx, global_values: Optional[np.ndarray]) -> None:
    rows = fs.owned_row_index()
    if ctx is None or ctx.nranks == 1:
        f.host[rows] = global_values[fs.owned_global]
    elif ctx.rank == 0:
        gid_parts = ctx.gather_to_root(np.asarray(fs.owned_global, np.int64).tobytes())
        for peer in range(1, ctx.nranks):
            g = np.frombuffer(gid_parts[peer], dtype=np.int64)
            ctx.send(peer, _TAG_SCATTER, np.ascontiguousarray(global_values[g]).tobytes())
        f.host[rows] = global_values[fs.owned_global]
    else:
        ctx.gather_to_root(np.asarray(fs.owned_global, np.int64).tobytes())
        data = np.frombuffer(ctx.receive(0, _TAG_SCATTER), dtype=f.host.dtype)
        f.host[rows] = data.reshape(len(rows), f.levels)
    if f.state is MemoryState.SYNCED:
        f.state = MemoryState.HOST_DIRTY
