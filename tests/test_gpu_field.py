"""Field host/device mirror on real HBM: the reference's state machine and copy counters
(field.py:99-154, test_field.py:181-214) with real copies."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_round_trip_and_counters(gpu):
    sg = gpu
    f = sg.create_field("f", (1000, 137))
    f.host[:] = np.random.default_rng(1).normal(size=f.host.shape)
    keep = f.host.copy()
    f.allocate_device()
    assert f.state is sg.MemoryState.SYNCED and f.copy_counters["host_to_device"] == 1
    assert np.array_equal(f.device.to_numpy(), keep)
    with f.device_view(sg.Intent.READ_WRITE):
        pass
    assert f.state is sg.MemoryState.DEVICE_DIRTY
    f.host[:] = 0
    f.update_host()
    assert np.array_equal(f.host, keep) and f.copy_counters["device_to_host"] == 1
    with f.host_view(sg.Intent.READ_WRITE) as h:
        h[0, 0] = 42.0
    assert f.state is sg.MemoryState.HOST_DIRTY
    f.syncHostDevice()
    assert f.state is sg.MemoryState.SYNCED and f.device.to_numpy()[0, 0] == 42.0
    with pytest.raises(sg.AlreadyAllocated):
        f.allocate_device()


@pytest.mark.parametrize("kind", ["REAL64", "REAL32", "INT32", "INT64"])
@pytest.mark.parametrize("levels", [1, 3, 16, 137])
def test_kinds_and_pitches(gpu, kind, levels):
    sg = gpu
    k = getattr(sg.Kind, kind)
    f = sg.create_field("f", (257, levels), k)
    f.host[:] = (np.arange(257 * levels).reshape(257, levels) % 1000).astype(k.dtype)
    f.allocate_device()
    assert f.device.pitch >= levels
    assert np.array_equal(f.device.to_numpy(), f.host)
    rows = f.device.download_rows(100, 50)
    assert np.array_equal(rows, f.host[100:150])


def test_cuda_array_interface(gpu):
    sg = gpu
    f = sg.create_field("f", (10, 137)).allocate_device()
    cai = f.device.__cuda_array_interface__
    assert cai["shape"] == (10, 137) and cai["strides"][0] == f.device.pitch * 8
    torch = pytest.importorskip("torch")
    t = torch.as_tensor(f.device, device="cuda")
    assert t.shape == (10, 137)


def test_stale_reads_raise(gpu):
    sg = gpu
    f = sg.create_field("f", (4, 2))
    with pytest.raises(sg.NoDevice):
        f.device_view()
    f.allocate_device()
    with f.host_view(sg.Intent.READ_WRITE):
        pass
    with pytest.raises(sg.StaleDevice):
        f.device_view()
    f.update_device()
    with f.device_view(sg.Intent.READ_WRITE):
        pass
    with pytest.raises(sg.StaleHost):
        f.host_view()


def test_pinned_registration_context(gpu):
    sg = gpu
    f = sg.create_field("f", (5000, 137))
    f.host[:] = np.random.default_rng(3).normal(size=f.host.shape)
    with sg.pinned(f.host):
        f.allocate_device()
    assert np.array_equal(f.device.to_numpy(), f.host)
    with sg.pinned(f.host):  # registering again after unregistering works
        pass


def test_create_field_pins_large_host_mirrors(gpu):
    """Host mirrors >= PIN_HOST_BYTES are page-locked, mapped and zero-filled (np.zeros
    semantics), so apply_remap on host fields can use the GPU gather; small ones stay numpy."""
    sg = gpu
    from paper_1908_07038_b200 import field as F
    from paper_1908_07038_b200.interp import _is_pinned

    rows = F.PIN_HOST_BYTES // (8 * 137) + 1
    big = sg.create_field("big", (rows, 137))
    assert _is_pinned(big.host) and big.host.shape == (rows, 137) and big.host.dtype == np.float64
    assert not big.host.any()
    small = sg.create_field("small", (100, 137))
    assert not _is_pinned(small.host) and not small.host.any()
    i32 = sg.create_field("i32", (F.PIN_HOST_BYTES // 4 + 7, 1), sg.Kind.INT32)
    assert _is_pinned(i32.host) and i32.host.dtype == np.int32 and not i32.host.any()
    big.host[-1, -1] = 3.0  # writable, and round-trips through the device like any mirror
    big.allocate_device()
    assert big.device.to_numpy()[-1, -1] == 3.0
    with big.device_view(sg.Intent.READ_WRITE):
        pass
    big.host[:] = 0
    big.update_host()
    assert big.host[-1, -1] == 3.0


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("dtype,levels", [(np.float64, 137), (np.float32, 3), (np.int32, 1), (np.int64, 5)])
def test_upload_row_runs(gpu, pinned, dtype, levels):
    """sg_field_h2d_row_runs: only the listed row runs change on the device (one DMA per run
    from pageable memory, one pull kernel from pinned mapped memory when there are many)."""
    sg = gpu
    from paper_1908_07038_b200.device import DeviceArray, PinnedArray

    n = 5000
    rng = np.random.default_rng(levels)
    src = PinnedArray((n, levels), dtype).array if pinned else np.empty((n, levels), dtype)
    src[:] = rng.integers(-1000, 1000, size=(n, levels)).astype(dtype)
    d = DeviceArray(n, levels, dtype)
    base = np.full((n, levels), 7, dtype)
    d.upload(base)
    starts = np.sort(rng.choice(n - 10, 60, replace=False))
    starts = starts[np.concatenate([[True], np.diff(starts) > 10])]
    runs = np.stack([starts, rng.integers(0, 10, len(starts))], axis=1)
    d.upload_row_runs(src, runs)
    expect = base.copy()
    for r0, k in runs:
        expect[r0:r0 + k] = src[r0:r0 + k]
    assert np.array_equal(d.to_numpy(), expect)
    from paper_1908_07038_b200._native import NativeError

    with pytest.raises(NativeError):  # run past the last row: invalid argument, nothing copied
        d.upload_row_runs(src, np.array([[n - 1, 2]]))


def test_ensure_pinned_lifetime(gpu):
    """Plain numpy host arrays are registered once (mapped) and unregistered when the owning
    array dies; views, small arrays and overlapping ranges are left alone."""
    import gc

    from paper_1908_07038_b200 import device as D

    a = np.zeros((1 << 24,))  # 128 MiB
    assert not D.is_pinned(a)
    assert D.ensure_pinned(a) and D.is_pinned(a) and D.is_pinned(a[10:20])
    assert D.ensure_pinned(a)  # idempotent
    b = a[1:]  # overlapping, not contained: different range, already covered -> pinned
    assert D.is_pinned(b)
    small = np.zeros(100)
    assert not D.ensure_pinned(small)
    start = a.ctypes.data
    del a, b
    gc.collect()
    assert start not in D._pinned_ranges  # finalizer unregistered it
    c = np.zeros((1 << 24,))
    assert D.ensure_pinned(c)  # the range can be registered again (also if the address was reused)
    d = np.frombuffer(bytearray(1 << 27), dtype=np.float64)  # memory not owned by numpy
    assert not D.ensure_pinned(d)


def test_apply_remap_on_plain_numpy_fields_pins_them(gpu):
    """Field(host=np.zeros(...)) of >= 64 MiB: apply_remap registers the arrays and takes the
    GPU-gather path; results bitwise equal to the oracle."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200 import device as D

    S, T = sg.grid_from_name("O320"), sg.grid_from_name("O160")
    dist = sg.blocks_partition(S, 1)
    mesh = sg.generate_mesh(S, dist, 0, halo=2, include_pole=True)
    w = sg.build_remap(sg.NodeColumns(mesh, None), T, sg.matching_partition(T, S, dist))
    L = 160  # 421,122 x 160 x 8 B = 539 MB source, 138 MB target
    hs = np.random.default_rng(3).normal(size=(mesh.nb_nodes, L))
    src = sg.Field(name="s", shape=hs.shape, kind=sg.Kind.REAL64, host=hs)
    dst = sg.Field(name="d", shape=(len(w), L), kind=sg.Kind.REAL64, host=np.zeros((len(w), L)))
    sg.apply_remap(w, src, dst)
    assert D.is_pinned(src.host) and D.is_pinned(dst.host)
    assert np.array_equal(dst.host.view(np.uint64), O.apply_remap(w.nodes, w.weights, hs).view(np.uint64))
