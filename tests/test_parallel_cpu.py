"""Rank runtimes and the exchange-plan protocol on CPU: the thread runtime (run_ranks,
parallel.py:1-195 contract) and DistContext over torch.distributed/gloo with world_size
> 1, each building the reference's halo plans (checked against golden fixtures)."""
import os
import socket
import types

import numpy as np
import pytest

import paper_1908_07038_b200 as sg
from conftest import load_golden


def test_send_receive_tags_fifo_and_counters():
    def prog(ctx):
        if ctx.rank == 0:
            ctx.send(1, 7, b"a")
            ctx.send(1, 8, b"bb")
            ctx.send(1, 7, b"c")
            return ctx.messages_sent, ctx.bytes_sent
        got = [ctx.receive(0, 8), ctx.receive(0, 7), ctx.receive(0, 7)]
        return got, ctx.messages_received

    r = sg.run_ranks(2, prog)
    assert r[0] == (3, 4)
    assert r[1] == ([b"bb", b"a", b"c"], 3)


def test_deadlock_detected_and_unconsumed():
    with pytest.raises(sg.DeadlockDetected):
        sg.run_ranks(2, lambda ctx: ctx.receive(1 - ctx.rank, 1))
    with pytest.raises(sg.UnconsumedMessages):
        sg.run_ranks(2, lambda ctx: ctx.send(1, 3, b"x") if ctx.rank == 0 else None)
    with pytest.raises(sg.InvalidRank):
        sg.run_ranks(1, lambda ctx: ctx.send(0, 1, b""))


def test_gather_broadcast_barrier_share():
    def prog(ctx):
        parts = ctx.gather_to_root(bytes([ctx.rank]))
        b = ctx.broadcast_from_root(b"root" if ctx.rank == 0 else None)
        ctx.barrier()
        s = ctx.share(ctx.rank * 10)
        return parts, b, s

    r = sg.run_ranks(3, prog)
    assert r[0][0] == [b"\x00", b"\x01", b"\x02"] and r[1][0] is None
    assert all(x[1] == b"root" for x in r)
    assert all(x[2] == [0, 10, 20] for x in r)


def test_error_propagates():
    def prog(ctx):
        if ctx.rank == 1:
            raise ValueError("boom")
        ctx.receive(1, 5)

    with pytest.raises(ValueError):
        sg.run_ranks(2, prog)


@pytest.mark.parametrize("name,src", [("part_O32_O16_p4_h2", "O32"), ("part_F8_F4_p3_h1", "F8")])
def test_thread_plan_build_matches_reference(name, src):
    z = load_golden(name)
    S = sg.grid_with_latitudes(src, z["src_lat"])
    P, halo = int(z["nparts"]), int(z["halo"])

    def prog(ctx):
        mesh = sg.generate_mesh(S, sg.blocks_partition(S, ctx.nranks), ctx.rank, halo=halo, include_pole=True)
        plan = sg.NodeColumns(mesh, ctx).exchange_plan
        for p in range(ctx.nranks):
            assert (p in plan.send) == (f"r{ctx.rank}_send_{p}" in z)
            if p in plan.send:
                assert np.array_equal(plan.send[p], z[f"r{ctx.rank}_send_{p}"])
            if p in plan.recv:
                assert np.array_equal(plan.recv[p], z[f"r{ctx.rank}_recv_{p}"])
                # pull-kernel source rows: the owner's send list for us, in the same order
                assert len(plan.recv_remote[p]) == len(plan.recv[p])
        return plan, ctx.messages_sent

    res = sg.run_ranks(P, prog)
    for r, (plan, msgs) in enumerate(res):
        assert msgs == P - 1  # one request per other rank (functionspace.py:77-81)
        for p, rem in plan.recv_remote.items():
            assert np.array_equal(rem, res[p][0].send[r])


def test_inconsistent_mesh_detected():
    g = sg.grid_from_name("F8")

    def prog(ctx):
        mesh = sg.generate_mesh(g, sg.blocks_partition(g, 2), ctx.rank, halo=1, include_pole=True)
        if ctx.rank == 1:
            mesh.node_global[mesh.node_ghost] += 1  # ask for ids rank 0 does not own
            mesh.node_global[-1] = 10**6
        return sg.NodeColumns(mesh, ctx)

    with pytest.raises(sg.InconsistentMesh):
        sg.run_ranks(2, prog)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = load_golden("part_F8_F4_p3_h1")
        S = sg.grid_with_latitudes("F8", z["src_lat"])
        ctx = sg.DistContext()
        mesh = sg.generate_mesh(S, sg.blocks_partition(S, world), rank, halo=int(z["halo"]), include_pole=True)
        plan = sg.NodeColumns(mesh, ctx).exchange_plan
        ok = all(np.array_equal(plan.send[p], z[f"r{rank}_send_{p}"]) for p in plan.send)
        ok &= all(np.array_equal(plan.recv[p], z[f"r{rank}_recv_{p}"]) for p in plan.recv)
        ok &= set(plan.send) == {p for p in range(world) if f"r{rank}_send_{p}" in z}
        gathered = ctx.gather_to_root(bytes([rank]))
        b = ctx.broadcast_from_root(b"xy" if rank == 0 else None)
        shared = ctx.share(rank + 100)
        q.put((rank, bool(ok), ctx.messages_sent, gathered, b, shared))
        ctx.barrier()
    finally:
        dist.destroy_process_group()


def test_distcontext_gloo_world3_plan_build():
    import torch.multiprocessing as mp

    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(o[1] for o in out)
    assert out[0][3] == [b"\x00", b"\x01", b"\x02"]
    assert all(o[4] == b"xy" for o in out)
    assert all(o[5] == [100, 101, 102] for o in out)


def test_send_runs_cover_the_union_of_send_lists():
    """HaloExchangePlan.send_runs: ascending (row0, nrows) runs of the union of every peer's
    send list — the rows the host-field halo_exchange stages on the device."""
    from paper_1908_07038_b200.functionspace import HaloExchangePlan

    rng = np.random.default_rng(0)
    send = {p: rng.choice(5000, 700, replace=False).astype(np.int64) for p in (1, 3, 6)}
    plan = HaloExchangePlan(nnodes=6000, send=send)
    runs = plan.send_runs()
    assert runs.dtype == np.int64 and (runs[:, 1] > 0).all()
    covered = np.concatenate([np.arange(r0, r0 + n) for r0, n in runs])
    assert np.array_equal(covered, np.unique(np.concatenate(list(send.values()))))
    assert (runs[1:, 0] > runs[:-1, 0] + runs[:-1, 1]).all()  # maximal runs: gaps between them
    assert HaloExchangePlan(nnodes=10).send_runs().shape == (0, 2)


def test_create_field_without_gpu_is_plain_numpy():
    """No device: create_field keeps np.zeros host storage at any size (no pinning attempt)."""
    import paper_1908_07038_b200 as sg
    from paper_1908_07038_b200 import field as F

    if sg._native.device_count() > 0:
        pytest.skip("a GPU is present")
    f = sg.create_field("x", (F.PIN_HOST_BYTES // 8 + 1, 1))
    assert isinstance(f.host, np.ndarray) and f.host.base is None and not f.host.any()


class _FakeArray:
    def __init__(self, ptr, handle):
        self.ptr, self.handle, self.device = ptr, handle, 0


def _gloo_signal_worker(rank, world, port, q, same_gpu):
    """The collective decisions behind the signalled exchange (parallel._signalled_exchange):
    ranks agree on signalled vs host-barrier mode from the device UUIDs, and on cache reuse,
    even when one rank's field buffer changes between calls (the ADVICE r1 hazard)."""
    import torch.distributed as dist

    import paper_1908_07038_b200._native as N
    import paper_1908_07038_b200.execute as E
    import paper_1908_07038_b200.parallel as PAR

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N.device_uuid = lambda dev: b"one-gpu" if same_gpu else bytes([rank]) * 16
        built = []

        class FakeExchange:
            @classmethod
            def for_rank(cls, ctx, plan, field):
                ctx.share(("build", field.ptr))  # collective, like peer_fields / peer_signals
                built.append(field.ptr)
                return cls()

        E.SignalledExchange = FakeExchange
        ctx = sg.DistContext(device=0)
        plan = types.SimpleNamespace(peers=[1 - rank])
        a, b = _FakeArray(1000 + rank, 1), _FakeArray(2000 + rank, 2)
        seq = [a, a, b if rank == 1 else a, a, a]
        got = [PAR._signalled_exchange(ctx, plan, x) for x in seq]
        q.put((rank, [g is None for g in got], built))
        ctx.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("same_gpu", [False, True])
def test_signalled_exchange_decisions_are_collective(same_gpu):
    import torch.multiprocessing as mp

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_signal_worker, args=(r, world, port, q, same_gpu)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    if same_gpu:  # spinning launches must not wait on each other on one GPU: never signalled
        assert all(o[1] == [True] * 5 and o[2] == [] for o in out)
    else:
        assert all(o[1] == [False] * 5 for o in out)
        # call 1 builds; call 3 rebuilds on BOTH ranks because rank 1's buffer changed
        assert [len(o[2]) for o in out] == [2, 2]
        assert out[1][2] == [1001, 2001] and out[0][2] == [1000, 1000]


def test_dist_context_keeps_every_peer_mapping_until_close(monkeypatch):
    """DistContext's CUDA-IPC mapping cache (host logic, no GPU): each (peer, handle, device)
    is opened once; sharing a NEW buffer of a peer never unmaps an older one that a built step
    or exchange may still point into; close_ipc unmaps everything exactly once."""
    import ctypes

    from paper_1908_07038_b200 import _native as N
    from paper_1908_07038_b200.parallel import DistContext

    calls = []
    nxt = iter(range(0x1000, 0x100000, 0x1000))

    def fake_call(name, *args):
        calls.append(name)
        if name == "sg_ipc_open":  # (device, handle address, 64, out-pointer address)
            ctypes.c_uint64.from_address(args[3]).value = next(nxt)
        elif name == "sg_ipc_close":
            closed.append(args[1])
        else:
            raise AssertionError(name)

    closed = []
    monkeypatch.setattr(N, "call", fake_call)
    ctx = DistContext.__new__(DistContext)  # only the cache logic: no process group needed
    ctx._ipc, ctx._ipc_sig = {}, {}
    a1 = DistContext._ipc_map(ctx._ipc, 1, b"A" * 64, 0)
    a1_again = DistContext._ipc_map(ctx._ipc, 1, b"A" * 64, 0)
    b1 = DistContext._ipc_map(ctx._ipc, 1, b"B" * 64, 0)  # peer 1 shares another buffer
    a2 = DistContext._ipc_map(ctx._ipc, 2, b"A" * 64, 0)  # same bytes from another peer: own key
    s1 = DistContext._ipc_map(ctx._ipc_sig, 1, b"S" * 64, 0)
    assert a1 == a1_again and len({a1, b1, a2, s1}) == 4
    assert calls.count("sg_ipc_open") == 4 and not closed  # nothing unmapped while in use
    ctx.close_ipc()
    assert sorted(closed) == sorted([a1, b1, a2, s1]) and not ctx._ipc and not ctx._ipc_sig


def _gloo_ipc_fail_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1908_07038_b200._native as N
    import paper_1908_07038_b200.parallel as PAR

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def fake_call(name, *args):
            if name == "sg_ipc_handle":
                return None
            raise AssertionError(name)

        N.call = fake_call

        def failing_map(cache, r, blob, device):
            if rank == 1:
                raise RuntimeError("cudaIpcOpenMemHandle: peer access unsupported")
            return 0x1000 + r

        PAR.DistContext._ipc_map = staticmethod(failing_map)
        ctx = sg.DistContext(device=0)
        arr = _FakeArray(0x5000 + rank, 1)
        arr.pitch = 137
        try:
            ctx.peer_fields(arr)
            outcome = "returned"
        except sg.SpheregridError as exc:
            outcome = "raised: " + str(exc)
        after = ctx.share(rank)  # the next collective still lines up on both ranks
        q.put((rank, outcome, after))
        ctx.barrier()
    except Exception as exc:  # noqa: BLE001 - reported to the test instead of a queue timeout
        q.put((rank, "error: " + repr(exc), None))
    finally:
        dist.destroy_process_group()


def test_peer_mapping_failure_raises_on_every_rank():
    """An IPC mapping that fails on ONE rank makes every rank raise (DistContext._all_or_none),
    so no rank enters the next collective alone — the N>1 bench then falls back to NCCL
    together instead of hanging."""
    import torch.multiprocessing as mp

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_ipc_fail_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(o[1].startswith("raised") and "rank 1" in o[1] for o in out), out
    assert all(o[2] == [0, 1] for o in out)
