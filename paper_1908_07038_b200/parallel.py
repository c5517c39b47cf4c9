"""Rank runtimes: the communication backend under NodeColumns / halo_exchange.

``run_ranks`` / ``RankContext`` keep the reference's in-process model and contract
(parallel.py:1-195): N rank programs on N threads, blocking tagged FIFO send/receive per
(source, destination), barrier, gather/broadcast through rank 0, deadlock detection, an
unconsumed-message check and the messages_sent / bytes_sent / messages_received counters
the reference's tests assert.  B200 additions: every rank thread is pinned to a GPU
(``devices``, default: the visible GPUs round-robin, else device 0), and ranks of one
process share device pointers through ``share`` so the device halo exchange is a single
pull kernel over peer memory (same device, or NVLink P2P) — no host staging.

``DistContext`` is the same interface over ``torch.distributed`` for one process per GPU
(torchrun): host messages on a gloo group, device halo exchange through the library's own
NCCL communicator (grouped ncclSend/ncclRecv between pack and unpack kernels).
"""

from __future__ import annotations

import pickle
import threading
from collections import deque
from dataclasses import dataclass, field
from typing import Any, Callable, Dict, List, Optional

from . import device as D
from .errors import DeadlockDetected, InvalidRank, UnconsumedMessages

_GATHER_TAG = 1 << 20  # parallel.py:19
_BCAST_TAG = (1 << 20) + 1  # parallel.py:20


class _Abort(Exception):
    """Another rank failed; unwind quietly."""


class _World:
    def __init__(self, nranks: int):
        self.nranks = nranks
        self.cv = threading.Condition()
        self.boxes: Dict[tuple, deque] = {}
        self.waiting: Dict[int, Callable[[], bool]] = {}
        self.done: set = set()
        self.deadlocked = False
        self.aborted = False
        self.epoch = 0
        self.arrived = 0
        self.board: Dict[tuple, Any] = {}

    def box(self, src: int, dst: int) -> deque:
        return self.boxes.setdefault((src, dst), deque())

    def _stuck(self) -> bool:
        # every unfinished rank waits and nobody's wake-up condition holds (parallel.py:49-64)
        if self.aborted:
            return False
        live = self.nranks - len(self.done)
        return live > 0 and len(self.waiting) == live and not any(p() for p in self.waiting.values())

    def block(self, rank: int, ready: Callable[[], bool]) -> None:
        self.waiting[rank] = ready
        try:
            if self._stuck():
                self.deadlocked = True
                self.cv.notify_all()
            while not ready():
                if self.aborted:
                    raise _Abort()
                if self.deadlocked:
                    raise DeadlockDetected(f"rank {rank} blocked with no possible sender")
                self.cv.wait()
        finally:
            self.waiting.pop(rank, None)

    def finish(self, rank: int) -> None:
        self.done.add(rank)
        if self._stuck():
            self.deadlocked = True
        self.cv.notify_all()


@dataclass
class RankContext:
    rank: int
    nranks: int
    _rt: _World = field(repr=False, default=None)
    messages_sent: int = 0
    bytes_sent: int = 0
    messages_received: int = 0
    device: int = 0
    _share_seq: int = field(repr=False, default=0)

    def _peer(self, peer: int) -> None:
        if not isinstance(peer, int) or not 0 <= peer < self.nranks:
            raise InvalidRank(f"rank {peer} not in [0, {self.nranks})")
        if peer == self.rank:
            raise InvalidRank("self-send/receive not allowed")

    def send(self, dest: int, tag: int, payload: bytes) -> None:
        self._peer(dest)
        data = bytes(payload)
        w = self._rt
        with w.cv:
            w.box(self.rank, dest).append((tag, data))
            self.messages_sent += 1
            self.bytes_sent += len(data)
            w.cv.notify_all()

    def receive(self, source: int, tag: int) -> bytes:
        self._peer(source)
        w = self._rt
        with w.cv:
            q = w.box(source, self.rank)

            def find():
                return next((k for k, (t, _) in enumerate(q) if t == tag), None)

            if find() is None:
                w.block(self.rank, lambda: find() is not None)
            k = find()
            _, data = q[k]
            del q[k]
            self.messages_received += 1
            return data

    def barrier(self) -> None:
        w = self._rt
        with w.cv:
            epoch = w.epoch
            w.arrived += 1
            if w.arrived == w.nranks:
                w.epoch += 1
                w.arrived = 0
                w.cv.notify_all()
                return
            w.block(self.rank, lambda: w.epoch > epoch)

    def gather_to_root(self, payload: bytes) -> Optional[List[bytes]]:
        if self.rank != 0:
            self.send(0, _GATHER_TAG, payload)
            return None
        return [bytes(payload)] + [self.receive(s, _GATHER_TAG) for s in range(1, self.nranks)]

    def broadcast_from_root(self, payload: Optional[bytes]) -> bytes:
        if self.rank != 0:
            return self.receive(0, _BCAST_TAG)
        data = bytes(payload)
        for d in range(1, self.nranks):
            self.send(d, _BCAST_TAG, data)
        return data

    # -- B200 additions ---------------------------------------------------------------------
    def share(self, value: Any) -> List[Any]:
        """Collective: every rank contributes ``value``; all get the list ordered by rank.
        Not a message (no counters): ranks of one process share an address space."""
        self._share_seq += 1
        key = self._share_seq
        w = self._rt
        with w.cv:
            w.board[(key, self.rank)] = value
        self.barrier()
        with w.cv:
            out = [w.board[(key, r)] for r in range(self.nranks)]
        self.barrier()
        with w.cv:
            w.board.pop((key, self.rank), None)
        return out

    def peer_fields(self, dev_array, plan=None) -> list:
        """(ptr, pitch, device) of every rank's instance of a field.  Collective, on every
        call: each rank may pass a different buffer from call to call (its field's mirror or
        a staging copy, depending on that rank's field state), so nothing is cached that a
        peer could have replaced.  With ``plan``, the ranks' send lists travel along (by
        reference: one address space) and complete a plan that lacks owner rows."""
        got = self.share((dev_array.ptr, dev_array.pitch, dev_array.device, plan.send if plan is not None else None))
        if plan is not None:
            plan.complete_remote(self.rank, {r: g[3] for r, g in enumerate(got) if r != self.rank})
        enabled = self.__dict__.setdefault("_p2p", set())
        for _, _, dev, _ in got:  # NVLink P2P between this rank's GPU and every peer's
            if dev != dev_array.device and (dev_array.device, dev) not in enabled:
                from . import _native as N

                N.call("sg_enable_peer_access", dev_array.device, dev)
                enabled.add((dev_array.device, dev))
        return [g[:3] for g in got]

    def peer_signals(self, signal) -> list:
        """(signal words pointer, device uuid) of every rank's step signal (execute.Signal).
        Collective.  One address space: raw device pointers (NVLink P2P between GPUs, enabled
        by peer_fields)."""
        from . import _native as N

        return self.share((signal.ptr, N.device_uuid(signal.device)))

    def device_exchange(self, plan, dev_array, stream: int = 0) -> None:
        """Device halo exchange over peer memory.  Every rank on its own GPU: one signalled
        pull kernel per rank (owners' ready words, no host barrier).  Ranks sharing a GPU: one
        pull kernel per rank between two host barriers (owners' rows final before, not
        overwritten while peers read)."""
        x = _signalled_exchange(self, plan, dev_array)
        if x is not None:
            x.launch(stream)
            D.synchronize(dev_array.device, stream)
            x.check()
            return
        ptrs = self.peer_fields(dev_array, plan)
        D.synchronize(dev_array.device, stream)
        self.barrier()
        plan.pull(dev_array, ptrs, stream)
        D.synchronize(dev_array.device, stream)
        self.barrier()


def _signalled_exchange(ctx, plan, dev_array):
    """The signalled pull exchange (execute.SignalledExchange) of ``plan`` on ``dev_array`` when
    every rank drives its own GPU, else None.  Collective on every call (ranks decide together
    whether to reuse their cached objects, so a rank whose field buffer changed never leaves
    the others in a different collective); at most 4 cached objects per rank, FIFO."""
    from . import _native as N
    from .execute import SignalledExchange

    cache = ctx.__dict__.setdefault("_xcache", [])
    key = (id(plan), dev_array.ptr, dev_array.handle)
    hit = next((x for k, x in cache if k == key), None)
    from .execute import MAX_SIGNAL_PEERS

    everyone = ctx.share((hit is not None, N.device_uuid(dev_array.device), len(plan.peers) <= MAX_SIGNAL_PEERS))
    if len({u for _, u, _ in everyone}) != ctx.nranks or not all(f for _, _, f in everyone):
        return None  # ranks share a GPU (spinning launches must not wait on each other there), or too many peers
    if all(h for h, _, _ in everyone):
        return hit
    x = SignalledExchange.for_rank(ctx, plan, dev_array)
    cache.append((key, x))
    if len(cache) > 4:
        cache.pop(0)
    return x


def _default_devices() -> List[int]:
    from . import _native as N

    n = N.device_count()
    return list(range(n)) if n > 0 else [0]


def run_ranks(nranks: int, program: Callable[[RankContext], object], devices: Optional[List[int]] = None) -> list:
    """Run program(ctx) on nranks threads; results ordered by rank (parallel.py:154-195)."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    devs = list(devices) if devices is not None else None
    w = _World(nranks)
    results: list = [None] * nranks
    failures: list = [None] * nranks

    def body(r: int) -> None:
        ctx = RankContext(rank=r, nranks=nranks, _rt=w)
        try:
            if devs is None:
                dl = _default_devices()
            else:
                dl = devs
            ctx.device = dl[r % len(dl)]
            D.set_device(ctx.device)
            results[r] = program(ctx)
        except _Abort:
            pass
        except BaseException as exc:  # noqa: BLE001 - re-raised by the caller
            failures[r] = exc
            with w.cv:
                w.aborted = True
                w.cv.notify_all()
        finally:
            with w.cv:
                w.finish(r)

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for exc in failures:
        if exc is not None:
            raise exc
    left = sum(len(q) for q in w.boxes.values())
    if left:
        raise UnconsumedMessages(f"{left} messages left in queues at shutdown")
    return results


class DistContext:
    """RankContext contract over torch.distributed, one process per GPU.

    Host messages (plan build, gather) travel on a gloo group as uint8 tensors; counters
    mirror the reference.  ``device_exchange`` uses the library's NCCL communicator."""

    def __init__(self, group=None, device: Optional[int] = None, transport: str = "nvlink"):
        """transport: "nvlink" (default: one signalled pull kernel per rank over CUDA-IPC
        mappings of the owners' fields, owners' ready words instead of barriers; ranks that
        share a GPU fall back to "ipc"), "nccl" (pack -> grouped ncclSend/ncclRecv -> unpack,
        stream-ordered) or "ipc" (pull kernel over CUDA-IPC mappings between two host
        barriers; works for several processes on one GPU too)."""
        import torch.distributed as dist

        if transport not in ("nvlink", "nccl", "ipc"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        # CUDA-IPC mappings of peers' buffers, (peer rank, ipc handle bytes, device) -> mapped
        # pointer, kept until close_ipc: several objects (a remap's fused step, an exchange of
        # another field, ...) may use several of a peer's buffers at the same time, so a new
        # buffer never unmaps an old one that an existing kernel argument still points into
        self._ipc: Dict[tuple, int] = {}
        self._ipc_sig: Dict[tuple, int] = {}  # same, for the peers' step signal words
        self._dist = dist
        self.rank = dist.get_rank()
        self.nranks = dist.get_world_size()
        self._group = group if group is not None else (
            dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else None)
        self.device = D.current_device() if device is None else int(device)
        self.messages_sent = 0
        self.bytes_sent = 0
        self.messages_received = 0
        self._comm = None
        self._pending: Dict[tuple, deque] = {}
        self._inflight: list = []

    def _peer(self, peer: int) -> None:
        if not isinstance(peer, int) or not 0 <= peer < self.nranks:
            raise InvalidRank(f"rank {peer} not in [0, {self.nranks})")
        if peer == self.rank:
            raise InvalidRank("self-send/receive not allowed")

    def send(self, dest: int, tag: int, payload: bytes) -> None:
        import torch

        self._peer(dest)
        data = pickle.dumps((tag, bytes(payload)))
        n = torch.tensor([len(data)], dtype=torch.int64)
        body = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        # non-blocking: the reference protocol sends to every peer before receiving
        # (functionspace.py:77-93); a blocking gloo send would deadlock it
        works = [self._dist.isend(n, dest, group=self._group), self._dist.isend(body, dest, group=self._group)]
        self._inflight.append((works, n, body))
        self._inflight = [w for w in self._inflight if not all(x.is_completed() for x in w[0])]
        self.messages_sent += 1
        self.bytes_sent += len(payload)

    def receive(self, source: int, tag: int) -> bytes:
        import torch

        self._peer(source)
        q = self._pending.setdefault(source, deque())
        while True:
            for k, (t, data) in enumerate(q):
                if t == tag:
                    del q[k]
                    self.messages_received += 1
                    return data
            n = torch.zeros(1, dtype=torch.int64)
            self._dist.recv(n, source, group=self._group)
            buf = torch.empty(int(n.item()), dtype=torch.uint8)
            self._dist.recv(buf, source, group=self._group)
            q.append(pickle.loads(buf.numpy().tobytes()))

    def flush(self) -> None:
        for works, _, _ in self._inflight:
            for w in works:
                w.wait()
        self._inflight = []

    def barrier(self) -> None:
        self.flush()
        self._dist.barrier(group=self._group)

    def gather_to_root(self, payload: bytes) -> Optional[List[bytes]]:
        if self.rank != 0:
            self.send(0, _GATHER_TAG, payload)
            return None
        return [bytes(payload)] + [self.receive(s, _GATHER_TAG) for s in range(1, self.nranks)]

    def broadcast_from_root(self, payload: Optional[bytes]) -> bytes:
        if self.rank != 0:
            return self.receive(0, _BCAST_TAG)
        data = bytes(payload)
        for d in range(1, self.nranks):
            self.send(d, _BCAST_TAG, data)
        return data

    def share(self, value: Any) -> List[Any]:
        self.flush()
        out: List[Any] = [None] * self.nranks
        self._dist.all_gather_object(out, value, group=self._group)
        return out

    def nccl_comm(self) -> int:
        if self._comm is None:
            import ctypes as C

            from . import _native as N

            uid = (C.c_uint8 * 128)()
            if self.rank == 0:
                N.call("sg_nccl_unique_id", N.ref(uid), 128)
            blob = self.share(bytes(uid) if self.rank == 0 else None)[0]
            uid = (C.c_uint8 * 128).from_buffer_copy(blob)
            h = C.c_uint64(0)
            N.call("sg_comm_create", self.device, self.nranks, self.rank, N.ref(uid), 128, N.ref(h))
            self._comm = N.Handle(h.value)
        return self._comm.handle

    def comm_info(self) -> dict:
        """NCCL's own view of this rank's communicator (sg_comm_info)."""
        import ctypes as C

        from . import _native as N

        v = [C.c_int32(0) for _ in range(4)]
        N.call("sg_comm_info", self.nccl_comm(), *[N.ref(x) for x in v])
        return {"nranks": v[0].value, "rank": v[1].value, "device": v[2].value, "nccl_version": v[3].value}

    @staticmethod
    def _ipc_map(cache: Dict[tuple, int], r: int, blob: bytes, device: int) -> int:
        """This process's mapping of peer r's buffer with IPC handle ``blob`` (opened once)."""
        import ctypes as C

        from . import _native as N

        key = (r, blob, device)
        ptr = cache.get(key)
        if ptr is None:
            p = C.c_uint64(0)
            hb = (C.c_uint8 * 64).from_buffer_copy(blob)
            N.call("sg_ipc_open", device, N.ref(hb), 64, N.ref(p))
            ptr = cache[key] = p.value
        return ptr

    def peer_fields(self, dev_array, plan=None) -> list:
        """(ptr, pitch, device) of every rank's copy of this field, via CUDA IPC.  Collective
        on every call (each rank may pass a different buffer per call); each peer buffer is
        mapped once and stays mapped until close_ipc, so objects built on earlier calls keep
        valid pointers.  Plans must carry their owner rows (``recv_remote``, set by
        build_exchange_plan)."""
        import ctypes as C

        from . import _native as N

        h = (C.c_uint8 * 64)()
        N.call("sg_ipc_handle", dev_array.handle, N.ref(h), 64)
        everyone = self.share((bytes(h), dev_array.pitch, dev_array.device))

        def mapped():
            return [(dev_array.ptr, dev_array.pitch, dev_array.device) if r == self.rank else
                    (self._ipc_map(self._ipc, r, blob, dev_array.device), pitch, dev)
                    for r, (blob, pitch, dev) in enumerate(everyone)]

        return self._all_or_none(mapped)

    def _all_or_none(self, local_step):
        """Run a rank-local step that may fail (opening CUDA-IPC mappings), then agree: if it
        failed on ANY rank every rank raises the same error class, so no rank goes on to the
        next collective while another has left (which would hang the job)."""
        from .errors import SpheregridError

        try:
            out, err = local_step(), ""
        except Exception as exc:  # noqa: BLE001 - reported collectively below
            out, err = None, f"rank {self.rank}: {exc}"
        errs = [e for e in self.share(err) if e]
        if errs:
            raise SpheregridError("CUDA-IPC mapping of peer memory failed (" + "; ".join(errs) + ")")
        return out

    def peer_signals(self, signal) -> list:
        """(pointer to rank r's step signal words, mapped here through CUDA IPC, device uuid)
        for every rank.  Collective; each peer signal is mapped once, until close_ipc."""
        import ctypes as C

        from . import _native as N

        h = (C.c_uint8 * 64)()
        N.call("sg_signal_ipc_handle", signal.handle, N.ref(h), 64)
        everyone = self.share((bytes(h), N.device_uuid(signal.device)))
        return self._all_or_none(lambda: [
            (signal.ptr, uuid) if r == self.rank else (self._ipc_map(self._ipc_sig, r, blob, signal.device), uuid)
            for r, (blob, uuid) in enumerate(everyone)])

    def close_ipc(self) -> None:
        """Unmap every peer field and step signal opened through CUDA IPC (call when no kernel
        that uses them is pending: after the last step / exchange of this context)."""
        from . import _native as N

        for (_, _, dev), ptr in list(self._ipc.items()) + list(self._ipc_sig.items()):
            N.call("sg_ipc_close", dev, ptr)
        self._ipc.clear()
        self._ipc_sig.clear()

    def device_exchange(self, plan, dev_array, stream: int = 0) -> None:
        if self.transport == "nccl":
            plan.exchange_nccl(dev_array, self.nccl_comm(), stream)
            D.synchronize(dev_array.device, stream)
            return
        if self.transport == "nvlink":
            x = _signalled_exchange(self, plan, dev_array)
            if x is not None:
                x.launch(stream)
                D.synchronize(dev_array.device, stream)
                x.check()
                return
        peers = self.peer_fields(dev_array)
        D.synchronize(dev_array.device, stream)
        self.barrier()  # every owner's rows are final
        plan.pull(dev_array, peers, stream)
        D.synchronize(dev_array.device, stream)
        self.barrier()  # nobody overwrites owned rows while a peer still reads them
