"""The distributed execute: halo exchange of the source field + apply, per rank (the
steady-state loop of run_remap_pipeline, cli.py:137-144, with the field kept in HBM).

Targets whose three stencil nodes are all owned rows (local rows < n_owned) do not need
the exchange: the largest contiguous block of them is applied on the main stream while the
exchange (pack -> grouped NCCL send/recv -> unpack) runs on a second stream; the remaining
(boundary) targets follow once the exchange's event fires.  With ``capture()`` the whole step
is recorded into one CUDA graph and replayed per call.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from . import _native as N
from .device import DeviceArray, Event, Graph, Stream
from .interp import APPLY_DEFAULT, InterpolationWeights, apply_remap_fused, apply_remap_range


def interior_block(weights: InterpolationWeights, n_owned: int):
    """[b0, b1): the longest run of targets whose stencil touches owned rows only."""
    inside = (weights.nodes < n_owned).all(axis=1)
    if not inside.any():
        return 0, 0
    d = np.diff(np.concatenate([[0], inside.astype(np.int8), [0]]))
    starts, ends = np.flatnonzero(d == 1), np.flatnonzero(d == -1)
    k = int(np.argmax(ends - starts))
    return int(starts[k]), int(ends[k])


class DistributedRemap:
    def __init__(self, fs, weights: InterpolationWeights, ctx, src: DeviceArray, dst: DeviceArray,
                 variant: int = APPLY_DEFAULT, overlap: bool = True, fused: bool = False):
        """fused: skip the ghost copy — boundary targets read ghost rows straight from the
        owners' fields (sg_remap_apply_fused; peer memory: in-process ranks or CUDA IPC).
        The source field's ghost rows are then left untouched."""
        self.fs, self.w, self.ctx = fs, weights, ctx
        self.src, self.dst = src, dst
        self.variant = variant
        self.plan = fs.exchange_plan
        self.m = len(weights)
        self.n_owned = fs.mesh.nb_owned_nodes
        self.b0, self.b1 = interior_block(weights, self.n_owned) if overlap else (0, 0)
        dev = src.device
        self.main = Stream(dev)
        self.halo = Stream(dev)
        self.ev_fork, self.ev_halo = Event(dev), Event(dev)
        self.graph: Optional[Graph] = None
        self.multi = ctx is not None and getattr(ctx, "nranks", 1) > 1
        # NCCL: stream-ordered exchange, overlappable and graph-capturable.  Otherwise
        # (in-process ranks, CUDA-IPC pull) the exchange is host-synchronised: no overlap.
        self.stream_ordered = self.multi and getattr(ctx, "transport", None) == "nccl"
        self.fused = bool(fused) and self.multi
        # fused + NCCL: peer pointers from CUDA IPC (NVLink reads), fenced by stream-ordered
        # NCCL barriers -> no host round trip and graph-capturable; fused without NCCL
        # (in-process ranks, IPC transport) fences with host barriers
        self.comm = ctx.nccl_comm() if self.stream_ordered else None
        self.peer_info = ctx.peer_fields(src) if self.fused else None

    @property
    def launches_per_step(self) -> int:
        n = 0
        if self.fused:
            return sum(1 for a, b in ((self.b0, self.b1), (0, self.b0), (self.b1, self.m)) if b > a)
        if self.multi and not self.stream_ordered:
            return 1 + int(sum(len(v) for v in self.plan.recv.values()) > 0)  # pull + apply
        if self.multi:
            n += int(sum(len(v) for v in self.plan.send.values()) > 0)  # pack
            n += int(sum(len(v) for v in self.plan.recv.values()) > 0)  # unpack
        ranges = [(self.b0, self.b1), (0, self.b0), (self.b1, self.m)]
        return n + sum(1 for a, b in ranges if b > a)

    def _enqueue(self) -> None:
        main = self.main.stream
        if self.fused:
            def fence():
                if self.stream_ordered:
                    N.call("sg_comm_barrier", self.comm, main)
                else:
                    self.main.synchronize()
                    self.ctx.barrier()

            if self.b1 > self.b0 and self.stream_ordered:  # interior rows need no fence
                apply_remap_range(self.w, [self.src], [self.dst], self.b0, self.b1, self.variant, main)
            fence()  # every owner's rows are final
            if self.b1 > self.b0 and not self.stream_ordered:
                apply_remap_range(self.w, [self.src], [self.dst], self.b0, self.b1, self.variant, main)
            for a, b in ((0, self.b0), (self.b1, self.m)):
                if b > a:
                    apply_remap_fused(self.w, self.plan, self.src, self.dst, a, b, self.peer_info, main)
            fence()  # nobody overwrites owned rows while a peer still reads them
            return
        if self.multi and not self.stream_ordered:
            self.main.synchronize()
            self.ctx.device_exchange(self.plan, self.src)
            apply_remap_range(self.w, [self.src], [self.dst], 0, self.m, self.variant, main)
            return
        if self.multi:
            self.ev_fork.record(main)
            self.halo.wait(self.ev_fork)
            self.plan.exchange_nccl(self.src, self.comm, self.halo.stream)
            self.ev_halo.record(self.halo.stream)
        if self.b1 > self.b0:
            apply_remap_range(self.w, [self.src], [self.dst], self.b0, self.b1, self.variant, main)
        if self.multi:
            self.main.wait(self.ev_halo)
        for a, b in ((0, self.b0), (self.b1, self.m)):
            if b > a:
                apply_remap_range(self.w, [self.src], [self.dst], a, b, self.variant, main)

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
