"""Per-thread device selection and device arrays.

One host thread drives one GPU (the run_ranks model, SURVEY.md §5 "distributed comm
backend"): ``set_device`` pins the calling thread's device; fields allocated afterwards
live there.  ``DeviceArray`` is a pitched (npts, levels) view of a library-owned field
buffer; it exports ``__cuda_array_interface__`` so torch / cupy can wrap it zero-copy.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from . import _native as N

_tls = threading.local()


def set_device(device: int) -> None:
    _tls.device = int(device)


def current_device() -> int:
    return getattr(_tls, "device", 0)


def synchronize(device: int = None, stream: int = 0) -> None:
    N.call("sg_stream_synchronize", current_device() if device is None else device, stream)


class DeviceArray(N.Handle):
    """Library-owned device buffer of one field (Field.device, field.py:102 of the
    reference is a numpy copy; here it is HBM)."""

    __slots__ = ("device", "shape", "dtype", "pitch", "ptr")

    def __init__(self, npts: int, levels: int, dtype: np.dtype, device: int = None):
        dev = current_device() if device is None else device
        h, pitch, p = C.c_uint64(0), C.c_int64(0), C.c_uint64(0)
        dtype = np.dtype(dtype)
        N.call("sg_field_alloc", dev, npts, levels, dtype.itemsize, N.ref(h), N.ref(pitch), N.ref(p))
        super().__init__(h.value)
        self.device = dev
        self.shape = (int(npts), int(levels))
        self.dtype = dtype
        self.pitch = pitch.value  # elements
        self.ptr = p.value

    @property
    def __cuda_array_interface__(self):
        typestr = self.dtype.str
        return {
            "shape": self.shape,
            "typestr": typestr,
            "data": (self.ptr, False),
            "strides": (self.pitch * self.dtype.itemsize, self.dtype.itemsize),
            "version": 3,
        }

    def upload(self, host: np.ndarray, stream: int = 0, sync: bool = True) -> None:
        if host.shape != self.shape or host.dtype != self.dtype or not host.flags["C_CONTIGUOUS"]:
            raise ValueError("host array must be C-contiguous with the field's shape and kind")
        N.call("sg_field_h2d", self.handle, N.ptr(host), stream)
        if sync:
            synchronize(self.device, stream)

    def download(self, host: np.ndarray, stream: int = 0, sync: bool = True) -> None:
        if host.shape != self.shape or host.dtype != self.dtype or not host.flags["C_CONTIGUOUS"]:
            raise ValueError("host array must be C-contiguous with the field's shape and kind")
        N.call("sg_field_d2h", self.handle, N.ptr(host), stream)
        if sync:
            synchronize(self.device, stream)

    def upload_rows(self, row0: int, host_rows: np.ndarray, stream: int = 0, sync: bool = True) -> None:
        host_rows = np.ascontiguousarray(host_rows, dtype=self.dtype)
        N.call("sg_field_h2d_rows", self.handle, row0, len(host_rows), N.ptr(host_rows), stream)
        if sync:
            synchronize(self.device, stream)

    def upload_row_runs(self, host: np.ndarray, runs: np.ndarray, stream: int = 0, sync: bool = True) -> None:
        """Rows ``[r0, r0 + n)`` of the full host array ``host`` for every (r0, n) in ``runs``
        into the same device rows."""
        if host.shape != self.shape or host.dtype != self.dtype or not host.flags["C_CONTIGUOUS"]:
            raise ValueError("host array must be C-contiguous with the device array's shape and dtype")
        runs = np.ascontiguousarray(runs, dtype=np.int64).reshape(-1, 2)
        N.call("sg_field_h2d_row_runs", self.handle, N.ptr(runs), len(runs), N.ptr(host), stream)
        if sync:
            synchronize(self.device, stream)

    def download_rows_into(self, row0: int, out: np.ndarray, stream: int = 0) -> None:
        """Rows ``[row0, row0 + len(out))`` into the C-contiguous host array ``out``."""
        if out.ndim != 2 or out.shape[1] != self.shape[1] or out.dtype != self.dtype or not out.flags["C_CONTIGUOUS"]:
            raise ValueError("out must be C-contiguous (rows, levels) of the device array's dtype")
        N.call("sg_field_d2h_rows", self.handle, row0, len(out), N.ptr(out), stream)
        synchronize(self.device, stream)

    def download_rows(self, row0: int, nrows: int, stream: int = 0) -> np.ndarray:
        out = np.empty((nrows, self.shape[1]), dtype=self.dtype)
        N.call("sg_field_d2h_rows", self.handle, row0, nrows, N.ptr(out), stream)
        synchronize(self.device, stream)
        return out

    def to_numpy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        self.download(out)
        return out

    # -- numpy-compatible access (the reference's Field.device was an ndarray, field.py:102) --
    # Element access moves data over PCIe; it exists so code written against the reference's
    # device mirror keeps working.  Kernels and torch/cupy use __cuda_array_interface__.
    @property
    def ndim(self) -> int:
        return 2

    @property
    def size(self) -> int:
        return self.shape[0] * self.shape[1]

    def __len__(self) -> int:
        return self.shape[0]

    def __array__(self, dtype=None, copy=None):
        a = self.to_numpy()
        return a if dtype is None else a.astype(dtype)

    def tobytes(self) -> bytes:
        return self.to_numpy().tobytes()

    def __getitem__(self, key):
        return self.to_numpy()[key]

    def __setitem__(self, key, value):
        if isinstance(key, slice) and key == slice(None):
            full = np.empty(self.shape, dtype=self.dtype)
            full[...] = np.asarray(value)
        else:
            full = self.to_numpy()
            full[key] = np.asarray(value)
        self.upload(np.ascontiguousarray(full))

    def _np(self, other):
        return np.asarray(other) if isinstance(other, DeviceArray) else other

    def __eq__(self, other):
        return self.to_numpy() == self._np(other)

    def __ne__(self, other):
        return self.to_numpy() != self._np(other)

    def __lt__(self, other):
        return self.to_numpy() < self._np(other)

    def __le__(self, other):
        return self.to_numpy() <= self._np(other)

    def __gt__(self, other):
        return self.to_numpy() > self._np(other)

    def __ge__(self, other):
        return self.to_numpy() >= self._np(other)

    def __add__(self, other):
        return self.to_numpy() + self._np(other)

    __radd__ = __add__

    def __sub__(self, other):
        return self.to_numpy() - self._np(other)

    def __rsub__(self, other):
        return self._np(other) - self.to_numpy()

    def __mul__(self, other):
        return self.to_numpy() * self._np(other)

    __rmul__ = __mul__

    def __truediv__(self, other):
        return self.to_numpy() / self._np(other)

    def __neg__(self):
        return -self.to_numpy()

    __hash__ = N.Handle.__hash__


class PinnedArray:
    """Page-locked host array (cudaHostAlloc) for full-rate asynchronous copies."""

    def __init__(self, shape, dtype=np.float64, write_combined: bool = False, zero: bool = False):
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        p = C.c_uint64(0)
        N.call("sg_host_alloc_flags", nbytes, int(bool(write_combined)) | (2 if zero else 0), N.ref(p))
        self._ptr = p.value
        buf = (C.c_char * max(nbytes, 1)).from_address(self._ptr)
        buf._sg_owner = self  # any view of .array keeps the pinned allocation alive
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self) -> None:
        if self._ptr:
            self.array = None
            if not N._shutting_down:
                N.call("sg_host_free", self._ptr)
            self._ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Event(N.Handle):
    """CUDA event on a device; ``elapsed_ms(start, end)`` synchronises on ``end``."""

    __slots__ = ()

    def __init__(self, device: int = None):
        h = C.c_uint64(0)
        N.call("sg_event_create", current_device() if device is None else device, N.ref(h))
        super().__init__(h.value)

    def record(self, stream: int = 0) -> "Event":
        N.call("sg_event_record", self.handle, stream)
        return self

    @staticmethod
    def elapsed_ms(start: "Event", end: "Event") -> float:
        ms = C.c_float(0)
        N.call("sg_event_elapsed_ms", start.handle, end.handle, N.ref(ms))
        return float(ms.value)


class Stream(N.Handle):
    """A non-blocking CUDA stream owned by the library; ``.stream`` is the raw handle every
    sg_* call accepts."""

    __slots__ = ("device", "stream")

    def __init__(self, device: int = None):
        dev = current_device() if device is None else device
        h, s = C.c_uint64(0), C.c_uint64(0)
        N.call("sg_stream_create", dev, N.ref(h), N.ref(s))
        super().__init__(h.value)
        self.device, self.stream = dev, s.value

    def wait(self, event: "Event") -> None:
        N.call("sg_stream_wait_event", self.stream, event.handle)

    def synchronize(self) -> None:
        synchronize(self.device, self.stream)


class Graph(N.Handle):
    """A captured sequence of stream work (cudaStreamBeginCapture ... EndCapture),
    instantiated once and replayed with ``launch``."""

    __slots__ = ("device",)

    def __init__(self, device: int, stream: int, body):
        N.call("sg_graph_begin", device, stream)
        try:
            body()
        finally:
            h = C.c_uint64(0)
            N.call("sg_graph_end", device, stream, N.ref(h))
        super().__init__(h.value)
        self.device = device

    def launch(self, stream: int) -> None:
        N.call("sg_graph_launch", self.handle, stream)


class pinned:
    """Context manager page-locking existing host arrays (cudaHostRegister) for the duration:
    ``with pinned(f.host, tf.host): apply_remap(w, f, tf)`` runs the host-buffer execute at
    full PCIe rate without copying into a PinnedArray."""

    def __init__(self, *arrays: np.ndarray):
        self.arrays = [a for a in arrays if a is not None and a.nbytes]
        self._done: list = []

    def __enter__(self):
        for a in self.arrays:
            if not a.flags["C_CONTIGUOUS"]:
                raise ValueError("only C-contiguous arrays can be registered")
            N.call("sg_host_register", a.ctypes.data, a.nbytes)
            self._done.append(a)
        return self

    def __exit__(self, *exc):
        for a in self._done:
            N.call("sg_host_unregister", a.ctypes.data)
        self._done = []
        return False


# ---- page-locking user arrays for the host-field execute paths --------------------------
# Host fields built on plain numpy arrays (Field(host=...)) would otherwise go through the
# driver's pageable staging copies (apply_remap at cfg3: 270 ms instead of 116 ms,
# profiles/r01_e2e_modes.md).  Large arrays are registered (cudaHostRegister, mapped) the first
# time a host-field path sees them and stay registered for the life of the numpy array that
# owns the memory: a weakref finalizer unregisters them when that array is deallocated (numpy
# clears weak references before it frees the data).
AUTO_PIN_BYTES = 64 << 20
_pin_lock = threading.Lock()
_pinned_ranges: dict = {}  # start address -> (end address, finalizer)


def _owner(a: np.ndarray):
    base = a
    while isinstance(base, np.ndarray) and base.base is not None:
        base = base.base
    return base


def is_pinned(a: np.ndarray) -> bool:
    """True when ``a`` lies in a library pinned allocation (PinnedArray) or in a range
    registered by :func:`ensure_pinned`."""
    own = _owner(a)
    if isinstance(getattr(own, "_sg_owner", None), PinnedArray):
        return True
    lo, hi = a.ctypes.data, a.ctypes.data + a.nbytes
    with _pin_lock:
        return any(s <= lo and hi <= e for s, (e, _) in _pinned_ranges.items())


def _unregister(start: int) -> None:
    with _pin_lock:
        _pinned_ranges.pop(start, None)
    if not N._shutting_down:
        try:
            N.call("sg_host_unregister", start)
        except Exception:  # noqa: BLE001 - context already gone at interpreter exit
            pass


def ensure_pinned(a: np.ndarray, min_bytes: int = AUTO_PIN_BYTES) -> bool:
    """Page-lock ``a`` in place (if it is large, C-contiguous and owned by a numpy array) for
    the rest of the owning array's life.  Returns whether ``a`` is pinned afterwards."""
    if a is None or a.nbytes == 0:
        return False
    if is_pinned(a):
        return True
    if a.nbytes < min_bytes or not a.flags["C_CONTIGUOUS"] or N.device_count() < 1:
        return False
    own = _owner(a)
    if not isinstance(own, np.ndarray) or not own.flags["OWNDATA"]:
        return False  # memory owned by something we cannot watch (mmap, buffer object)
    start, end = a.ctypes.data, a.ctypes.data + a.nbytes
    with _pin_lock:
        if any(s < end and start < e for s, (e, _) in _pinned_ranges.items()):
            return False  # overlaps another registration (a different view of the same data)
        try:
            N.call("sg_host_register", start, a.nbytes)
        except Exception:  # noqa: BLE001 - not registrable (e.g. out of lockable memory)
            return False
        _pinned_ranges[start] = (end, weakref.finalize(own, _unregister, start))
    return True
