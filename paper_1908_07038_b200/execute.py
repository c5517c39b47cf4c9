"""The distributed execute: halo exchange of the source field + apply, per rank (the
steady-state loop of run_remap_pipeline, cli.py:137-144, with the field kept in HBM).

Targets whose stencil nodes are all owned rows (local rows < n_owned) do not need the
exchange ("interior"); the others ("boundary") do.  With a stream-ordered transport (NCCL)
the interior targets are applied on the main stream while the exchange (pack -> grouped
NCCL send/recv -> unpack) runs on a second stream; the boundary targets follow once the
exchange's event fires.  Both sets are device target lists, so any decomposition (bands or
equal regions, whose boundary targets interleave with interior ones) overlaps fully.  With
``fused=True`` there is no ghost copy at all: boundary targets read ghost rows straight from
their owners' fields inside the apply kernel (sg_remap_apply_fused_list), fenced by NCCL
barriers (stream-ordered) or host barriers.  ``capture()`` records a stream-ordered step into
one CUDA graph.
"""

from __future__ import annotations

from typing import Optional

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
        self.stream_ordered = self.multi and getattr(ctx, "transport", None) == "nccl"
        self.fused = bool(fused) and self.multi
        self.comm = ctx.nccl_comm() if self.stream_ordered else None
        self.peer_info = ctx.peer_fields(src, self.plan) if self.fused else None

    @property
    def launches_per_step(self) -> int:
        applies = int(self.interior is not None) + int(self.boundary is not None)
        if not self.multi:
            return 1
        if self.fused:
            return applies
        if not self.stream_ordered:
            return 1 + int(sum(len(v) for v in self.plan.recv.values()) > 0)  # pull + apply
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
        if self.fused:
            def fence():
                if self.stream_ordered:
                    N.call("sg_comm_barrier", self.comm, main)
                else:
                    self.main.synchronize()
                    self.ctx.barrier()

            if self.stream_ordered:  # interior rows are local: no fence needed before them
                self._apply(self.interior, main)
            fence()  # every owner's rows are final
            if not self.stream_ordered:
                self._apply(self.interior, main)
            if self.boundary is not None:
                apply_remap_fused_list(self.w, self.plan, self.src, self.dst, self.boundary, self.peer_info, main)
            fence()  # nobody overwrites owned rows while a peer still reads them
            return
        if not self.stream_ordered:
            self.main.synchronize()
            self.ctx.device_exchange(self.plan, self.src)
            apply_remap_range(self.w, [self.src], [self.dst], 0, self.m, self.variant, main)
            return
        self.ev_fork.record(main)
        self.halo.wait(self.ev_fork)
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
