"""ctypes binding of ``libsgb200.so`` (the C-ABI declared in include/spheregrid_b200.h).

There is no fallback: if the library is missing the import fails loudly and tells the user
to run ``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_1908_07038_b200/csrc``).  Status codes follow the reference's binding conventions
(frontend/src/errors.ts:7-16); domain errors are re-raised as the reference exception class
named in the message prefix.
"""

from __future__ import annotations

import ctypes as C
import os
import re
from typing import Optional

import numpy as np

from . import errors as E

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsgb200.so")


def _nccl_library() -> Optional[str]:
    """The NCCL the installed torch links (the nvidia-nccl wheel), so the library's lazy dlopen
    and a later ``import torch`` share one libnccl.so.2 (halo.cu nccl())."""
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (list(spec.submodule_search_locations or []) if spec else []):
        path = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(path):
            return path
    return None


if "SG_NCCL_LIBRARY" not in os.environ:
    _nccl = _nccl_library()
    if _nccl:
        os.environ["SG_NCCL_LIBRARY"] = _nccl

u64, i64, i32, u8p = C.c_uint64, C.c_int64, C.c_int32, C.POINTER(C.c_uint8)
vp, sz, dp = C.c_void_p, C.c_size_t, C.c_void_p

# name -> argtypes (all return int32 status)
_SIGS = {
    "sg_version": [C.c_char_p, sz],
    "sg_last_error": [C.c_char_p, sz],
    "sg_registry_count": [vp],
    "sg_release": [u64],
    "sg_device_count": [vp],
    "sg_device_uuid": [i32, vp, sz],
    "sg_stream_synchronize": [i32, u64],
    "sg_field_alloc": [i32, i64, i32, i32, vp, vp, vp],
    "sg_field_h2d": [u64, vp, u64],
    "sg_field_d2h": [u64, vp, u64],
    "sg_field_h2d_rows": [u64, i64, i64, vp, u64],
    "sg_field_d2h_rows": [u64, i64, i64, vp, u64],
    "sg_field_h2d_row_runs": [u64, vp, i64, vp, u64],
    "sg_field_info": [u64, vp, vp, vp, vp, vp],
    "sg_host_alloc": [sz, vp],
    "sg_host_alloc_flags": [sz, i32, vp],
    "sg_host_free": [u64],
    "sg_host_register": [u64, sz],
    "sg_host_unregister": [u64],
    "sg_event_create": [i32, vp],
    "sg_event_record": [u64, u64],
    "sg_event_elapsed_ms": [u64, u64, vp],
    "sg_stream_create": [i32, vp, vp],
    "sg_stream_wait_event": [u64, u64],
    "sg_enable_peer_access": [i32, i32],
    "sg_graph_begin": [i32, u64],
    "sg_graph_end": [i32, u64, vp],
    "sg_graph_launch": [u64, u64],
    "sg_locator_create": [i32, vp, i64, vp, vp, i64, vp],
    "sg_locator_stats": [u64, vp, vp, vp, vp],
    "sg_locator_locate": [u64, vp, i64, vp, vp],
    "sg_remap_build": [u64, vp, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp],
    "sg_stencil_create": [i32, vp, vp, i64, i64, vp],
    "sg_stencil_info": [u64, vp, vp, vp],
    "sg_stencil_create_k": [i32, vp, vp, i64, i32, i64, vp],
    "sg_bilinear_build": [i32, i32, vp, vp, i32, vp, i64, vp, i64, vp, vp, vp, vp, vp],
    "sg_remap_apply": [u64, vp, vp, i32, i32, u64],
    "sg_remap_apply_range": [u64, vp, vp, i32, i64, i64, i32, u64],
    "sg_remap_apply_list": [u64, vp, vp, i32, u64, i64, i32, u64],
    "sg_remap_execute_host": [u64, vp, vp, i32, vp, vp, i32, i32, i32, vp],
    "sg_halo_plan_create": [i32, i64, i32, vp, vp, vp, vp, vp, vp, vp],
    "sg_halo_plan_info": [u64, vp, vp],
    "sg_halo_pack": [u64, u64, vp, u64],
    "sg_halo_unpack": [u64, u64, vp, u64],
    "sg_halo_pull": [u64, u64, vp, vp, u64],
    "sg_remap_apply_fused": [u64, u64, u64, u64, i64, i64, vp, vp, u64],
    "sg_remap_apply_fused_list": [u64, u64, u64, u64, u64, i64, vp, vp, u64],
    "sg_nccl_unique_id": [vp, sz],
    "sg_comm_create": [i32, i32, i32, vp, sz, vp],
    "sg_halo_exchange_nccl": [u64, u64, u64, u64],
    "sg_comm_barrier": [u64, u64],
    "sg_comm_init_all": [i32, vp, vp],
    "sg_comm_info": [u64, vp, vp, vp, vp],
    "sg_field_checksum": [u64, i64, i64, vp, vp],
    "sg_rows_copy": [i32, u64, i64, u64, u64, i64, u64, i64, i64, u64],
    "sg_ipc_handle": [u64, vp, sz],
    "sg_ipc_open": [i32, vp, sz, vp],
    "sg_ipc_close": [i32, u64],
    "sg_signal_create": [i32, i32, i32, vp],
    "sg_signal_ptr": [u64, vp],
    "sg_signal_ipc_handle": [u64, vp, sz],
    "sg_signal_read": [u64, vp, i64],
    "sg_signal_write": [u64, vp, i64],
    "sg_step_create": [u64, u64, u64, u64, u64, vp, vp, vp, vp],
    "sg_step_info": [u64, vp, vp],
    "sg_step_launch": [vp, i32, i32, u64],
    "sg_step_launch_cooperative": [vp, i32, u64],
    "sg_step_check": [u64, vp, vp],
    "sg_step_set_timeout": [u64, u64],
    "sg_exchange_create": [u64, u64, u64, vp, vp, vp, vp],
    "sg_exchange_launch": [vp, i32, i32, u64],
    "sg_exchange_launch_cooperative": [vp, i32, u64],
    "sg_exchange_set_timeout": [u64, u64],
    "sg_exchange_signal": [u64, vp],
    "sg_meshgen_create": [i32, vp, i32, vp, i64, i32, i32, i32, vp, vp, vp, vp, vp],
    "sg_meshgen_fetch": [u64, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "sg_matching_partition": [i32, vp, vp, vp, vp, i64, i32, vp],
}

SG_OK, SG_DOMAIN_ERROR, SG_INVALID_HANDLE, SG_INVALID_ARGUMENT = 0, 1, 2, 3


class NativeError(E.SpheregridError):
    """Status 2/3 from the C-ABI (invalid handle / argument)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def _load() -> C.CDLL:
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"native library {_LIB_PATH} is missing: build it with "
            "`make -C paper_1908_07038_b200/csrc` (there is no CPU fallback)"
        )
    lib = C.CDLL(_LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int32
    return lib


lib = _load()
_shutting_down = False


def _mark_shutdown() -> None:
    # registered after the CUDA runtime's own exit handlers, so it runs first: from here on
    # handles are leaked to the OS instead of released into a runtime being torn down
    global _shutting_down
    _shutting_down = True


import atexit  # noqa: E402

atexit.register(_mark_shutdown)
_PREFIX = re.compile(r"^([A-Za-z]+): (.*)$", re.S)


def last_error() -> str:
    buf = C.create_string_buffer(2048)
    lib.sg_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int, **attrs) -> None:
    if status == SG_OK:
        return
    msg = last_error()
    if status == SG_DOMAIN_ERROR:
        m = _PREFIX.match(msg)
        if m:
            cls = E.error_class(m.group(1))
            if cls is E.NotLocated:
                raise E.NotLocated(m.group(2), target_global_index=attrs.get("target_global_index"))
            raise cls(m.group(2))
        raise E.SpheregridError(msg)
    raise NativeError(status, msg)


def call(name: str, *args, **attrs) -> None:
    check(getattr(lib, name)(*args), **attrs)


def ptr(a: Optional[np.ndarray]) -> Optional[int]:
    """Address of a C-contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data


def out_u64() -> C.c_uint64:
    return C.c_uint64(0)


def ref(x) -> int:
    return C.addressof(x)


def device_count() -> int:
    n = C.c_int32(0)
    call("sg_device_count", ref(n))
    return n.value


def device_uuid(device: int) -> bytes:
    buf = (C.c_uint8 * 16)()
    call("sg_device_uuid", device, ref(buf), 16)
    return bytes(buf)


def registry_count() -> int:
    n = C.c_int64(0)
    call("sg_registry_count", ref(n))
    return n.value


def release(handle: int) -> None:
    call("sg_release", handle)


def version() -> str:
    buf = C.create_string_buffer(256)
    call("sg_version", buf, len(buf))
    return buf.value.decode()


def exported_symbols() -> list:
    return sorted(_SIGS)


class Handle:
    """Owns one registry handle; released on close() or garbage collection."""

    __slots__ = ("handle",)

    def __init__(self, handle: int):
        self.handle = int(handle)

    def close(self) -> None:
        h, self.handle = self.handle, 0
        if h and not _shutting_down:
            lib.sg_release(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
