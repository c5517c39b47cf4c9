"""The distributed execute: halo exchange of the source field + apply, per rank (the
steady-state loop of run_remap_pipeline, cli.py:137-144, with the field kept in HBM).

Targets whose stencil nodes are all owned rows (local rows < n_owned) do not need the
exchange ("interior"); the others ("boundary") do.  With a stream-ordered transport (NCCL)
the interior targets are applied on the main stream while the exchange (pack -> grouped
NCCL send/recv -> unpack) runs on a second stream; the boundary targets follow once the
exchange's event fires.  Both sets are device target lists, so any decomposition (bands or
equal regions, whose boundary targets interleave with interior ones) overlaps fully.  With
``fused=True`` there is no ghost copy at all: boundary targets read ghost rows straight from
their owners' fields inside the apply kernel.  With one GPU per rank the fused step is ONE
kernel per rank (csrc/step.cu, ``FusedStep``): owners publish "rows final" and readers "done
reading" through flag words in each other's HBM (NVLink P2P / CUDA IPC), so no host or NCCL
barrier remains in the step.  Ranks sharing a GPU keep host barriers around the fused apply
(kernels that wait on each other must not be separate launches on one GPU); a single-GPU
emulation of P ranks runs every rank's step in one launch (``launch_fused_steps``).
``capture()`` records a stream-ordered step into one CUDA graph.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .device import DeviceArray, Event, Graph, Stream
from .interp import (APPLY_DEFAULT, InterpolationWeights, apply_remap_fused_list, apply_remap_list,
                     apply_remap_range)


def interior_block(weights: InterpolationWeights, n_owned: int):
    """[b0, b1): the longest run of targets whose stencil touches owned rows only."""
    inside = (weights.nodes < n_owned).all(axis=1)
    if not inside.any():
        return 0, 0
    d = np.diff(np.concatenate([[0], inside.astype(np.int8), [0]]))
    starts, ends = np.flatnonzero(d == 1), np.flatnonzero(d == -1)
    k = int(np.argmax(ends - starts))
    return int(starts[k]), int(ends[k])


def _device_list(rows: np.ndarray, device: int) -> Optional[DeviceArray]:
    if len(rows) == 0:
        return None
    d = DeviceArray(len(rows), 1, np.int32, device)
    d.upload(np.ascontiguousarray(rows.reshape(-1, 1), dtype=np.int32))
    return d


MAX_SIGNAL_PEERS = 16  # kPeers of csrc/step.cu: the peer table travels in the kernel parameters


class Signal(N.Handle):
    """A rank's step signal words in HBM (csrc/step.cu): ready[r], done[r], epoch, ..."""

    def __init__(self, device: int, nranks: int, rank: int):
        h = C.c_uint64(0)
        N.call("sg_signal_create", device, nranks, rank, N.ref(h))
        super().__init__(h.value)
        self.device, self.nranks, self.rank = device, nranks, rank
        p = C.c_uint64(0)
        N.call("sg_signal_ptr", self.handle, N.ref(p))
        self.ptr = p.value

    def check(self) -> int:
        """Raises if a device-side wait timed out; returns the last completed epoch."""
        w = self.read()
        if w["error"]:
            from .errors import SpheregridError

            raise SpheregridError(f"signalled launch of rank {self.rank} timed out waiting for a peer ("
                                  + ("owner rows never published" if w["error"] == 1 else "reader never finished")
                                  + ")")
        return w["epoch"]

    def publish_owners_ahead(self, epoch: int) -> None:
        """Measurement only: mark every rank's ready word as published up to ``epoch`` so this
        rank's launches run alone (one rank's step timed without its peers)."""
        w = np.zeros(2 * self.nranks + 4, np.uint64)
        N.call("sg_signal_read", self.handle, N.ptr(w), len(w))
        w[:self.nranks] = epoch
        N.call("sg_signal_write", self.handle, N.ptr(w), len(w))

    def read(self) -> dict:
        w = np.zeros(2 * self.nranks + 4, np.uint64)
        N.call("sg_signal_read", self.handle, N.ptr(w), len(w))
        R = self.nranks
        return {"ready": w[:R].tolist(), "done": w[R:2 * R].tolist(), "epoch": int(w[2 * R]),
                "current": int(w[2 * R + 1]), "count": int(w[2 * R + 2]), "error": int(w[2 * R + 3])}


class FusedStep(N.Handle):
    """One rank's exchange + apply as one kernel with device-side signalling
    (sg_step_create).  ``peer_info[r]`` = (ptr, pitch, device) of rank r's source field
    (ctx.peer_fields); ``peer_sigs[r]`` = (pointer to rank r's signal words, device uuid)
    (ctx.peer_signals).  Targets run in natural order; the ``n_boundary`` whose stencil reads
    a ghost row read it from the owner's field once the step's signal kernel has seen every
    owner's ready word."""

    def __init__(self, weights: InterpolationWeights, plan, src: DeviceArray, dst: DeviceArray, signal: Signal,
                 peer_info, peer_sigs):
        dev = src.device
        peers = plan.peers
        ptrs = np.array([peer_info[p][0] for p in peers] or [0], np.uint64)
        pitch = np.array([peer_info[p][1] for p in peers] or [0], np.int64)
        flags = np.array([peer_sigs[p][0] for p in peers] or [0], np.uint64)
        h = C.c_uint64(0)
        N.call("sg_step_create", weights.device_stencil(dev), plan.native(dev), src.handle, dst.handle, signal.handle,
               N.ptr(ptrs), N.ptr(pitch), N.ptr(flags), N.ref(h))
        super().__init__(h.value)
        self.signal, self.device = signal, dev
        m, nb = C.c_int64(0), C.c_int64(0)
        N.call("sg_step_info", self.handle, N.ref(m), N.ref(nb))
        self.m, self.n_boundary = m.value, nb.value
        self._keep = (weights, plan, src, dst)

    def launch(self, stream: int = 0) -> None:
        launch_fused_steps([self], stream, wait_done=True)

    def set_timeout(self, seconds: float) -> None:
        """Bound on every device-side wait of this step (default 10 s)."""
        N.call("sg_step_set_timeout", self.handle, max(1, int(seconds * 1e9)))

    def check(self) -> int:
        """Raises if a wait timed out; returns the last completed epoch (synchronous)."""
        err, ep = C.c_uint64(0), C.c_uint64(0)
        N.call("sg_step_check", self.handle, N.ref(err), N.ref(ep))
        return ep.value


def launch_fused_steps(steps: Sequence[FusedStep], stream: int = 0, wait_done: bool = False) -> None:
    """One signal kernel + one step kernel over the given ranks' steps (all on one device).
    Several ranks on one GPU: wait_done must be False (the host checks the words after)."""
    arr = np.array([s.handle for s in steps], np.uint64)
    N.call("sg_step_launch", N.ptr(arr), len(arr), int(bool(wait_done)), stream)


def launch_fused_steps_cooperative(steps: Sequence[FusedStep], stream: int = 0) -> None:
    """Every rank of a single-GPU emulation as ONE cooperative launch with the tail waits
    (wait_done): all blocks are co-resident, so each rank's finisher can wait for its readers'
    done words as it does with one GPU per rank.  Small problems only (the grid must fit)."""
    arr = np.array([s.handle for s in steps], np.uint64)
    N.call("sg_step_launch_cooperative", N.ptr(arr), len(arr), stream)


class DistributedRemap:
    def __init__(self, fs, weights: InterpolationWeights, ctx, src: DeviceArray, dst: DeviceArray,
                 variant: int = APPLY_DEFAULT, overlap: bool = True, fused: bool = False):
        self.fs, self.w, self.ctx = fs, weights, ctx
        self.src, self.dst = src, dst
        self.variant = variant
        self.plan = fs.exchange_plan
        self.m = len(weights)
        self.n_owned = fs.mesh.nb_owned_nodes
        dev = src.device
        inside = (weights.nodes < self.n_owned).all(axis=1) if overlap else np.zeros(self.m, bool)
        self.interior = _device_list(np.flatnonzero(inside), dev)
        self.boundary = _device_list(np.flatnonzero(~inside), dev)
        self.n_interior = int(inside.sum())
        self.main = Stream(dev)
        self.halo = Stream(dev)
        self.ev_fork, self.ev_halo = Event(dev), Event(dev)
        self.graph: Optional[Graph] = None
        self.multi = ctx is not None and getattr(ctx, "nranks", 1) > 1
        # NCCL: stream-ordered exchange, overlappable and graph-capturable.  Otherwise
        # (in-process ranks, CUDA-IPC pull) the exchange is host-synchronised: no overlap.
        self.fused = bool(fused) and self.multi
        transport = getattr(ctx, "transport", None)
        # not fused: the exchange is stream-ordered (and overlaps the interior targets) with NCCL
        # or, every rank on its own GPU, the signalled pull kernel (transport "nvlink")
        self.xchg = None
        if self.multi and not self.fused and transport == "nvlink":
            from .parallel import _signalled_exchange

            self.xchg = _signalled_exchange(ctx, self.plan, src)
        self.stream_ordered = self.multi and not self.fused and (transport == "nccl" or self.xchg is not None)
        self.comm = ctx.nccl_comm() if self.stream_ordered and self.xchg is None else None
        self.peer_info = ctx.peer_fields(src, self.plan) if self.fused else None
        # fused with one GPU per rank: device-side signalling, one kernel per rank per step.
        # The decision is collective (identical on every rank): every rank on its own GPU.
        self.signalled = False
        self.fused_step: Optional[FusedStep] = None
        if self.fused and hasattr(ctx, "peer_signals"):
            self.signal = Signal(dev, ctx.nranks, ctx.rank)
            sigs = ctx.peer_signals(self.signal)
            few = all(ctx.share(len(self.plan.peers) <= MAX_SIGNAL_PEERS))
            self.signalled = few and len({u for _, u in sigs}) == ctx.nranks
            if self.signalled:
                self.fused_step = FusedStep(weights, self.plan, src, dst, self.signal, self.peer_info, sigs)
                self.stream_ordered = True

    @property
    def launches_per_step(self) -> int:
        applies = int(self.interior is not None) + int(self.boundary is not None)
        if not self.multi:
            return 1
        if self.signalled:
            return 2  # signal kernel + step kernel
        if self.fused:
            return applies
        if not self.stream_ordered:
            return 1 + int(sum(len(v) for v in self.plan.recv.values()) > 0)  # pull + apply
        if self.xchg is not None:
            return 2 + applies  # signal + pull
        n = int(sum(len(v) for v in self.plan.send.values()) > 0)  # pack
        n += int(sum(len(v) for v in self.plan.recv.values()) > 0)  # unpack
        return n + applies

    def _apply(self, rows: Optional[DeviceArray], stream: int) -> None:
        if rows is not None:
            apply_remap_list(self.w, [self.src], [self.dst], rows, self.variant, stream)

    def _enqueue(self) -> None:
        main = self.main.stream
        if not self.multi:
            apply_remap_range(self.w, [self.src], [self.dst], 0, self.m, self.variant, main)
            return
        if self.signalled:
            self.fused_step.launch(main)
            return
        if self.fused:  # ranks share a GPU: host barriers around the peer reads
            self.main.synchronize()
            self.ctx.barrier()  # every owner's rows are final
            self._apply(self.interior, main)
            if self.boundary is not None:
                apply_remap_fused_list(self.w, self.plan, self.src, self.dst, self.boundary, self.peer_info, main)
            self.main.synchronize()
            self.ctx.barrier()  # nobody overwrites owned rows while a peer still reads them
            return
        if not self.stream_ordered:
            self.main.synchronize()
            self.ctx.device_exchange(self.plan, self.src)
            apply_remap_range(self.w, [self.src], [self.dst], 0, self.m, self.variant, main)
            return
        self.ev_fork.record(main)
        self.halo.wait(self.ev_fork)
        if self.xchg is not None:
            self.xchg.launch(self.halo.stream)
        else:
            self.plan.exchange_nccl(self.src, self.comm, self.halo.stream)
        self.ev_halo.record(self.halo.stream)
        self._apply(self.interior, main)  # overlaps the exchange
        self.main.wait(self.ev_halo)
        self._apply(self.boundary, main)

    def capture(self) -> None:
        """Record one step into a CUDA graph (call after one eager step so every buffer
        exists).  Only stream-ordered steps can be captured."""
        if self.multi and not self.stream_ordered:
            raise RuntimeError("a host-synchronised exchange cannot be captured")
        self.graph = Graph(self.src.device, self.main.stream, self._enqueue)

    def step(self) -> None:
        if self.graph is not None:
            self.graph.launch(self.main.stream)
        else:
            self._enqueue()

    def synchronize(self) -> None:
        self.main.synchronize()
        if self.fused_step is not None:
            self.fused_step.check()
        if self.xchg is not None:
            self.xchg.check()


def emulated_fused_steps(ranks: Sequence[tuple]) -> List[FusedStep]:
    """Fused steps of P ranks that all live on ONE GPU, for ``launch_fused_steps(steps)`` (one
    launch over every rank's data: the single-GPU stand-in for P GPUs).  ``ranks[r]`` =
    (weights, plan, src DeviceArray, dst DeviceArray) of rank r; plans need owner rows
    (build_exchange_plan sets them)."""
    P = len(ranks)
    dev = ranks[0][2].device
    if any(r[2].device != dev or r[3].device != dev for r in ranks):
        raise ValueError("an emulated launch needs every rank on one device")
    sigs = [Signal(dev, P, r) for r in range(P)]
    uuid = N.device_uuid(dev)
    peer_info = [(r[2].ptr, r[2].pitch, dev) for r in ranks]
    peer_sigs = [(s.ptr, uuid) for s in sigs]
    return [FusedStep(w, plan, src, dst, sigs[r], peer_info, peer_sigs)
            for r, (w, plan, src, dst) in enumerate(ranks)]


class SignalledExchange(N.Handle):
    """The halo exchange of ``plan`` on ``field`` (a DeviceArray) as one pull kernel per rank
    with device-side signalling (sg_exchange_create): every ghost row is copied from its
    owner's field once the owner published its epoch.  ``peer_info`` / ``peer_sigs`` as for
    FusedStep."""

    def __init__(self, plan, field: DeviceArray, signal: Signal, peer_info, peer_sigs):
        dev = field.device
        peers = plan.peers
        ptrs = np.array([peer_info[p][0] for p in peers] or [0], np.uint64)
        pitch = np.array([peer_info[p][1] for p in peers] or [0], np.int64)
        flags = np.array([peer_sigs[p][0] for p in peers] or [0], np.uint64)
        h = C.c_uint64(0)
        N.call("sg_exchange_create", plan.native(dev), field.handle, signal.handle, N.ptr(ptrs), N.ptr(pitch),
               N.ptr(flags), N.ref(h))
        super().__init__(h.value)
        self.signal, self.device = signal, dev
        self.nghosts = sum(len(v) for v in plan.recv.values())
        self._keep = (plan, field)

    def launch(self, stream: int = 0) -> None:
        launch_exchanges([self], stream, wait_done=True)

    def set_timeout(self, seconds: float) -> None:
        N.call("sg_exchange_set_timeout", self.handle, max(1, int(seconds * 1e9)))

    def check(self) -> int:
        return self.signal.check()

    @classmethod
    def for_rank(cls, ctx, plan, field: DeviceArray) -> "SignalledExchange":
        """Collective: every rank of ``ctx`` (all on distinct GPUs) builds its exchange."""
        info = ctx.peer_fields(field, plan)
        sig = Signal(field.device, ctx.nranks, ctx.rank)
        return cls(plan, field, sig, info, ctx.peer_signals(sig))


def launch_exchanges(xs: Sequence[SignalledExchange], stream: int = 0, wait_done: bool = False) -> None:
    arr = np.array([x.handle for x in xs], np.uint64)
    N.call("sg_exchange_launch", N.ptr(arr), len(arr), int(bool(wait_done)), stream)


def launch_exchanges_cooperative(xs: Sequence[SignalledExchange], stream: int = 0) -> None:
    """Cooperative single-GPU emulation of the exchange with the tail waits (see
    ``launch_fused_steps_cooperative``)."""
    arr = np.array([x.handle for x in xs], np.uint64)
    N.call("sg_exchange_launch_cooperative", N.ptr(arr), len(arr), stream)


def emulated_exchanges(ranks: Sequence[tuple]) -> List[SignalledExchange]:
    """Signalled exchanges of P ranks on ONE GPU, for one ``launch_exchanges(xs)``:
    ``ranks[r]`` = (plan, DeviceArray) of rank r."""
    P = len(ranks)
    dev = ranks[0][1].device
    if any(f.device != dev for _, f in ranks):
        raise ValueError("an emulated launch needs every rank on one device")
    sigs = [Signal(dev, P, r) for r in range(P)]
    uuid = N.device_uuid(dev)
    info = [(f.ptr, f.pitch, dev) for _, f in ranks]
    psig = [(s.ptr, uuid) for s in sigs]
    return [SignalledExchange(plan, f, sigs[r], info, psig) for r, (plan, f) in enumerate(ranks)]
