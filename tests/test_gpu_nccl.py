"""The NCCL plumbing on one GPU (a single-rank communicator): dlopen + symbol resolution,
unique id, communicator creation, grouped send/recv of an exchange with no peers, the
stream-ordered barrier, and capture of barrier + exchange + apply into a CUDA graph.  The
multi-rank exchange needs one GPU per rank (NCCL refuses two ranks on one device)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_single_rank_nccl_comm_barrier_and_graph(gpu):
    sg = gpu
    import paper_1908_07038_b200._native as N
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, Graph, Stream

    uid = (C.c_uint8 * 128)()
    N.call("sg_nccl_unique_id", N.ref(uid), 128)
    h = C.c_uint64(0)
    N.call("sg_comm_create", 0, 1, 0, N.ref(uid), 128, N.ref(h))
    comm = N.Handle(h.value)
    g, t = sg.grid_from_name("O32"), sg.grid_from_name("O16")
    dist = sg.blocks_partition(g, 1)
    mesh = sg.generate_mesh(g, dist, 0, halo=0, include_pole=True)
    fs = sg.NodeColumns(mesh, None)
    w = sg.build_remap(fs, t, sg.matching_partition(t, g, dist))
    hsrc = np.random.default_rng(2).normal(size=(mesh.nb_nodes, 7))
    src, dst = DeviceArray(mesh.nb_nodes, 7, np.float64), DeviceArray(len(w), 7, np.float64)
    src.upload(hsrc)
    st = Stream(0)
    plan = fs.exchange_plan
    plan.exchange_nccl(src, comm.handle, st.stream)  # no peers: pack/unpack skipped, empty group
    N.call("sg_comm_barrier", comm.handle, st.stream)
    st.synchronize()

    def body():
        N.call("sg_comm_barrier", comm.handle, st.stream)
        plan.exchange_nccl(src, comm.handle, st.stream)
        sg.apply_remap_device(w, [src], [dst], stream=st.stream)
        N.call("sg_comm_barrier", comm.handle, st.stream)

    graph = Graph(0, st.stream, body)
    for _ in range(3):
        graph.launch(st.stream)
    st.synchronize()
    exp = O.apply_remap(w.nodes, w.weights, hsrc)
    assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64))


def test_fork_join_capture_with_single_rank_nccl(gpu):
    """The multi-GPU step's graph shape: fork a second stream from the main stream with an
    event, run the (NCCL) exchange there while the main stream applies, join with a second
    event, then finish on the main stream — captured once and replayed."""
    sg = gpu
    import paper_1908_07038_b200._native as N
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, Event, Graph, Stream
    from paper_1908_07038_b200.interp import apply_remap_range

    uid = (C.c_uint8 * 128)()
    N.call("sg_nccl_unique_id", N.ref(uid), 128)
    h = C.c_uint64(0)
    N.call("sg_comm_create", 0, 1, 0, N.ref(uid), 128, N.ref(h))
    comm = N.Handle(h.value)
    g, t = sg.grid_from_name("O64"), sg.grid_from_name("O32")
    dist = sg.blocks_partition(g, 1)
    mesh = sg.generate_mesh(g, dist, 0, halo=0, include_pole=True)
    fs = sg.NodeColumns(mesh, None)
    w = sg.build_remap(fs, t, sg.matching_partition(t, g, dist))
    m = len(w)
    hsrc = np.random.default_rng(5).normal(size=(mesh.nb_nodes, 33))
    src, dst = DeviceArray(mesh.nb_nodes, 33, np.float64), DeviceArray(m, 33, np.float64)
    src.upload(hsrc)
    main, side = Stream(0), Stream(0)
    fork, join = Event(0), Event(0)
    fs.exchange_plan.exchange_nccl(src, comm.handle, side.stream)  # warm: buffers exist
    side.synchronize()

    def body():
        fork.record(main.stream)
        side.wait(fork)
        fs.exchange_plan.exchange_nccl(src, comm.handle, side.stream)
        N.call("sg_comm_barrier", comm.handle, side.stream)
        apply_remap_range(w, [src], [dst], 0, m // 3, 0, side.stream)
        join.record(side.stream)
        apply_remap_range(w, [src], [dst], m // 3, 2 * m // 3, 0, main.stream)
        main.wait(join)
        apply_remap_range(w, [src], [dst], 2 * m // 3, m, 0, main.stream)

    graph = Graph(0, main.stream, body)
    for _ in range(2):
        graph.launch(main.stream)
    main.synchronize()
    exp = O.apply_remap(w.nodes, w.weights, hsrc)
    assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64))


@pytest.mark.parametrize("dtype,levels", [(np.float64, 137), (np.float32, 5), (np.int64, 1)])
def test_nccl_self_exchange_payloads(gpu, dtype, levels):
    """Non-empty grouped ncclSend/ncclRecv through the real pack -> NCCL -> unpack path: a
    single-rank communicator whose plan sends rows to itself (NCCL allows self send/recv), so
    the payload offsets, pack order (requester's order) and unpack rows are exercised on one
    GPU.  ghost rows <- owner rows, bitwise."""
    sg = gpu
    import paper_1908_07038_b200._native as N
    from paper_1908_07038_b200.device import DeviceArray, Stream
    from paper_1908_07038_b200.functionspace import HaloExchangePlan

    uid = (C.c_uint8 * 128)()
    N.call("sg_nccl_unique_id", N.ref(uid), 128)
    h = C.c_uint64(0)
    N.call("sg_comm_create", 0, 1, 0, N.ref(uid), 128, N.ref(h))
    comm = N.Handle(h.value)
    n, nghost = 20000, 3000
    rng = np.random.default_rng(levels)
    owned = n - nghost
    send = rng.permutation(owned)[:nghost].astype(np.int64)  # permuted, like the reference's lists
    recv = np.arange(owned, n, dtype=np.int64)
    plan = HaloExchangePlan(nnodes=n, send={0: send}, recv={0: recv}, recv_remote={0: send})
    host = rng.integers(-10**6, 10**6, size=(n, levels)).astype(dtype)
    dev = DeviceArray(n, levels, dtype)
    dev.upload(host)
    st = Stream(0)
    plan.exchange_nccl(dev, comm.handle, st.stream)
    st.synchronize()
    expect = host.copy()
    expect[recv] = host[send]
    assert np.array_equal(dev.to_numpy(), expect)


def test_nccl_before_torch_import(gpu):
    """A fresh process that creates the library's NCCL communicator BEFORE importing torch can
    still import torch: the lazy dlopen loads the same libnccl.so.2 torch links
    (SG_NCCL_LIBRARY), not an older system NCCL under the same soname."""
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import ctypes as C, sys; sys.path.insert(0, %r)\n"
        "import paper_1908_07038_b200._native as N\n"
        "uid = (C.c_uint8 * 128)(); N.call('sg_nccl_unique_id', N.ref(uid), 128)\n"
        "h = C.c_uint64(0); N.call('sg_comm_create', 0, 1, 0, N.ref(uid), 128, N.ref(h))\n"
        "import torch; assert torch.cuda.is_available(); print('ok', torch.cuda.nccl.version())\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr[-2000:]


def test_comm_init_all_single_process(gpu):
    """sg_comm_init_all (ncclCommInitAll, one process driving its GPUs): the communicator of
    device 0 carries a real self-exchange and the stream-ordered barrier."""
    sg = gpu
    import paper_1908_07038_b200._native as N
    from paper_1908_07038_b200.device import DeviceArray, Stream
    from paper_1908_07038_b200.functionspace import HaloExchangePlan

    devs = np.array([0], np.int32)
    out = np.zeros(1, np.uint64)
    N.call("sg_comm_init_all", 1, N.ptr(devs), N.ptr(out))
    comm = N.Handle(int(out[0]))
    n, levels = 4000, 137
    rng = np.random.default_rng(11)
    send = rng.permutation(3000)[:1000].astype(np.int64)
    recv = np.arange(3000, n, dtype=np.int64)
    plan = HaloExchangePlan(nnodes=n, send={0: send}, recv={0: recv}, recv_remote={0: send})
    host = rng.normal(size=(n, levels))
    dev = DeviceArray(n, levels, np.float64)
    dev.upload(host)
    st = Stream(0)
    N.call("sg_comm_barrier", comm.handle, st.stream)
    plan.exchange_nccl(dev, comm.handle, st.stream)
    st.synchronize()
    expect = host.copy()
    expect[recv] = host[send]
    assert np.array_equal(dev.to_numpy(), expect)
