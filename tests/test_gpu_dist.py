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
