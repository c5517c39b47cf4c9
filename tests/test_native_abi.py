"""The C-ABI library loads, exports every symbol include/spheregrid_b200.h declares, and
follows the binding conventions (status codes, last error, never-reused handles)
— CPU only, no compute calls."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "spheregrid_b200.h")).read()
    return sorted(set(re.findall(r"^int32_t (sg_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_1908_07038_b200._native as N

    declared = header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(N.lib, name), name
    assert sorted(N.exported_symbols()) == declared


def test_library_is_built_for_sm100a():
    import subprocess

    import paper_1908_07038_b200._native as N

    out = subprocess.run(["cuobjdump", "--list-elf", N._LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_registry():
    import paper_1908_07038_b200._native as N

    assert "sm_100a" in N.version()
    assert N.registry_count() >= 0


def test_invalid_handle_and_double_release():
    import paper_1908_07038_b200._native as N

    assert N.lib.sg_release(987654321) == N.SG_INVALID_HANDLE
    assert "invalid handle" in N.last_error()
    # a meshgen handle is host-only: create, release, release again
    import numpy as np

    nl = np.array([4, 4], np.int64)
    part = np.zeros(8, np.int32)
    h = C.c_uint64(0)
    z = [C.c_int64(0) for _ in range(4)]
    before = N.registry_count()
    N.call("sg_meshgen_create", 2, N.ptr(nl), 0, N.ptr(part), 8, 1, 0, 0, N.ref(h), *[N.ref(x) for x in z])
    assert N.registry_count() == before + 1
    assert N.lib.sg_release(h.value) == N.SG_OK
    assert N.lib.sg_release(h.value) == N.SG_INVALID_HANDLE
    assert N.registry_count() == before
    h2 = C.c_uint64(0)
    N.call("sg_meshgen_create", 2, N.ptr(nl), 0, N.ptr(part), 8, 1, 0, 0, N.ref(h2), *[N.ref(x) for x in z])
    assert h2.value > h.value  # never reused
    N.release(h2.value)


def test_invalid_argument_status():
    import numpy as np

    import paper_1908_07038_b200._native as N

    nl = np.array([4, 4], np.int64)
    part = np.zeros(8, np.int32)
    h = C.c_uint64(0)
    z = [C.c_int64(0) for _ in range(4)]
    rc = N.lib.sg_meshgen_create(2, N.ptr(nl), 0, N.ptr(part), 8, 1, 3, 0, N.ref(h), *[N.ref(x) for x in z])
    assert rc == N.SG_INVALID_ARGUMENT
    assert "partition 3" in N.last_error()


def test_domain_error_maps_to_reference_class():
    import numpy as np

    import paper_1908_07038_b200 as sg
    import paper_1908_07038_b200._native as N

    nl = np.array([4, 4], np.int64)
    part = np.zeros(7, np.int32)
    h = C.c_uint64(0)
    z = [C.c_int64(0) for _ in range(4)]
    with pytest.raises(sg.InvalidDistribution):
        N.call("sg_meshgen_create", 2, N.ptr(nl), 0, N.ptr(part), 7, 1, 0, 0, N.ref(h), *[N.ref(x) for x in z])


def build_c_program(out_path):
    """tests/c_abi/remap_c.c: a plain C99 client of include/spheregrid_b200.h linked against
    libsgb200.so (what a non-Python binding compiles)."""
    import subprocess

    lib = os.path.join(ROOT, "paper_1908_07038_b200", "_lib")
    cmd = ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-Wall", "-Wextra", "-Werror",
           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c_abi", "remap_c.c"),
           "-o", str(out_path), "-L", lib, "-lsgb200", f"-Wl,-rpath,{lib}", "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out_path


def test_header_and_c_client_compile_and_link(tmp_path):
    """The header is valid C99 and every symbol the client uses resolves at link time."""
    exe = build_c_program(tmp_path / "remap_c")
    assert os.path.exists(exe)
