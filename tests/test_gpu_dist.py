"""One process per rank over torch.distributed (gloo host messages) with the device halo
exchange through CUDA-IPC mappings and the fused pull kernel.  Two processes share the one
GPU of the test box (IPC works within a device; the exchange is host-barrier synchronised,
no kernel waits on another)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1908_07038_b200 as sg

        sg.set_device(0)
        ctx = sg.DistContext(device=0, transport="ipc")
        g = sg.grid_from_name("O32")
        mesh = sg.generate_mesh(g, sg.blocks_partition(g, world), rank, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        f = fs.create_field("x", 137)
        owned = fs.owned_row_index()
        f.host[owned] = mesh.node_global[owned, None] * 1.0 + np.arange(137)[None, :] / 137
        f.allocate_device()
        fs.halo_exchange_device(f, ctx)
        f.update_host()
        ok = np.array_equal(f.host, mesh.node_global[:, None] * 1.0 + np.arange(137)[None, :] / 137)
        # host entry point through the same transport (staging copy)
        h = fs.create_field("y", 3, sg.Kind.INT64)
        h.host[owned] = mesh.node_global[owned, None]
        fs.halo_exchange(h, ctx)
        ok2 = np.array_equal(h.host, np.repeat(mesh.node_global[:, None], 3, axis=1))
        q.put((rank, bool(ok), bool(ok2), ctx.messages_sent))
        ctx.barrier()
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_pull_exchange_processes(gpu, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(o[1] and o[2] for o in out), out


@pytest.mark.parametrize("extra", [["--no-fused"], ["--fused"], ["--no-fused", "--transport", "nvlink"]])
def test_bench_torchrun_two_processes(gpu, extra):
    """The driver's N>1 launch line (torch.distributed.run, one process per rank) end to end on
    the one GPU of the test box: bench.py --gpus 2 with the CUDA-IPC transport on cfg2 (equal
    regions, halo 2) prints one JSON line with the multi-GPU keys (halo, roofline, e2e)."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--config", "cfg2"] + (extra if "--transport" in extra
                                                                     else ["--transport", "ipc"] + extra)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "strong"
    assert line["halo"]["bytes_per_exchange"] > 0 and line["roofline"]["bound"] == "hbm"
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["step"]["fused"] == ("--fused" in extra) and line["comm"]["transport_fallback"] is None
    assert line["step"]["device_signalled"] is False  # two ranks on one GPU: host barriers
    if "nvlink" in extra:  # signalled pulls need one GPU per rank: explicit host-barrier pull here
        assert line["comm"]["exchange"] == "pull kernel between host barriers"
    p = line["parity"]
    assert p["source_rows_bitwise"] and p["target_rows_bitwise"] and p["e2e_target_rows_bitwise"], p
    assert [h["halo"] for h in line["halo_sweep"]] == [1, 2, 3]
    assert all(h["ghosts_bitwise"] and h["bytes_per_exchange"] > 0 for h in line["halo_sweep"])
    b = [h["bytes_per_exchange"] for h in line["halo_sweep"]]
    assert b[0] < b[1] < b[2]


def _signal_worker(rank, world, port, q):
    """One rank of the signalled step / exchange with its peers' fields AND signal words mapped
    through CUDA IPC (DistContext.peer_fields / peer_signals), as with one GPU per rank.  Both
    processes share the test box's GPU, so no launch may wait for the other process: every
    epoch the owners' ready words are published ahead from the host and the tail wait is off
    (wait_done = 0).  What this proves across processes: IPC-mapped signal words (system
    scope) are written by the peer's kernels — ready by its signal kernel, done by its
    finisher — and ghost rows are read straight from the peer's field."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1908_07038_b200 as sg
        from oracle import oracle as O
        from paper_1908_07038_b200.device import DeviceArray, synchronize
        from paper_1908_07038_b200.execute import (FusedStep, Signal, SignalledExchange, launch_exchanges,
                                                   launch_fused_steps)

        sg.set_device(0)
        ctx = sg.DistContext(device=0, transport="ipc")
        S, T = sg.grid_from_name("O32"), sg.grid_from_name("O48")
        dist_s = sg.blocks_partition(S, world)
        mesh = sg.generate_mesh(S, dist_s, rank, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        plan = fs.exchange_plan
        w = sg.build_remap(fs, T, sg.matching_partition(T, S, dist_s), ctx)
        L = 300  # > 2 MB per field: separate allocations, not one sub-allocated block
        gvals = np.random.default_rng(44).normal(size=(S.npts + 2, L))
        init = np.where(mesh.node_ghost[:, None], 0.0, gvals[mesh.node_global])
        src, xf = DeviceArray(mesh.nb_nodes, L, np.float64), DeviceArray(mesh.nb_nodes, L, np.float64)
        src.upload(init)
        xf.upload(init)
        dst = DeviceArray(len(w), L, np.float64)
        sig, xsig = Signal(0, world, rank), Signal(0, world, rank)
        step = FusedStep(w, plan, src, dst, sig, ctx.peer_fields(src, plan), ctx.peer_signals(sig))
        x = SignalledExchange(plan, xf, xsig, ctx.peer_fields(xf, plan), ctx.peer_signals(xsig))
        # a third peer buffer and signal mapped AFTER the step and exchange were built: their
        # mappings of the peers' src / signal words must stay valid (large fields get their
        # own allocation, so an unmap would really unmap)
        other, osig = DeviceArray(mesh.nb_nodes, 512, np.float64), Signal(0, world, rank)
        ctx.peer_fields(other, plan)
        ctx.peer_signals(osig)
        epochs = 3
        for e in range(1, epochs + 1):
            sig.publish_owners_ahead(e)
            xsig.publish_owners_ahead(e)
            synchronize(0)
            ctx.barrier()  # every rank's rows final and no peer kernel in flight
            launch_exchanges([x], wait_done=False)
            launch_fused_steps([step], wait_done=False)
            synchronize(0)
            ctx.barrier()
        exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
        ok_step = bool(np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64)))
        ok_x = bool(np.array_equal(xf.to_numpy(), gvals[mesh.node_global]))
        ws, wx = sig.read(), xsig.read()
        done_ok = all(ws["done"][p] == epochs and wx["done"][p] == epochs for p in plan.send)
        words_ok = (ws["epoch"] == wx["epoch"] == epochs and ws["error"] == wx["error"] == 0
                    and ws["count"] == wx["count"] == 0)
        q.put((rank, ok_step, ok_x, bool(done_ok and words_ok), int(step.n_boundary), len(plan.send)))
        ctx.barrier()
        ctx.close_ipc()
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, False, False, repr(e), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_signalled_step_with_ipc_signals_across_processes(gpu, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_signal_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(o[1] and o[2] and o[3] for o in out), out
    assert sum(o[4] for o in out) > 0 and all(o[5] > 0 for o in out), out  # peer reads and readers exist
