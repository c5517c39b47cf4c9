"""The multi-GPU path across real devices: one process per GPU (torchrun), device halo
exchange through NCCL (pack -> grouped ncclSend/ncclRecv -> unpack) and the graph-captured,
overlapped step; ``bench.py`` checks every rank's exchanged source rows and target rows
bitwise against a single-process recomputation and reports NCCL's own rank count.  Needs
>= 2 visible GPUs (NCCL refuses two ranks on one device); skipped otherwise."""
import json
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ngpus():
    import paper_1908_07038_b200 as sg

    return sg._native.device_count()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("extra", [["--no-fused", "--transport", "nccl"], ["--fused", "--transport", "nccl"],
                                   ["--partitioner", "blocks", "--transport", "nccl"], ["--no-fused"], []])
def test_torchrun_nccl_two_gpus_bitwise(extra):
    if _ngpus() < 2:
        pytest.skip("needs >= 2 GPUs (one NCCL rank per device)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "5", "--warmup", "3", "--config", "cfg2"] + extra
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["comm"]["nccl_nranks"] == 2
    if "nccl" not in extra:  # default transport: the signalled NVLink pull, NCCL timed beside it
        assert line["comm"]["exchange"].startswith("signalled pull")
        assert all("nccl_baseline" in h and h["nccl_baseline"]["ghosts_bitwise"] for h in line["halo_sweep"])
    assert line["comm"]["transport_fallback"] is None
    # fused is the default: one kernel per rank with device-side signalling over NVLink
    assert line["step"]["device_signalled"] == ("--no-fused" not in extra)
    p = line["parity"]
    assert p["source_rows_bitwise"] and p["target_rows_bitwise"] and p["e2e_target_rows_bitwise"], p
    assert line["step"]["cuda_graph"] is True
    assert all(h["ghosts_bitwise"] for h in line["halo_sweep"])
