"""cfg4 halo-exchange sweep on ONE GPU (BASELINE configs[3] emulated): O1280, 137 levels,
P in {2,4,8}, halo 1..3.  All P ranks' fields live on device 0; each rank's exchange is
timed on its own (serialised) with CUDA events:
  * pull  — the fused kernel (pack + transfer + unpack in one pass over peer memory)
  * pack + unpack — the two kernels around the NCCL transfer of the multi-process path.
Bytes per exchange = Σ ghosts · L · 8 (SURVEY.md §8(d) halo metric).  Peer memory here is
the same HBM, so this measures the exchange kernels, not NVLink (NVLink needs >1 GPU).
Prints one JSON line per (P, halo)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg  # noqa: E402
from paper_1908_07038_b200.device import DeviceArray, Event  # noqa: E402

L = 137
REPS = 20


def main(grid="O1280", parts=(2, 4, 8), halos=(1, 2, 3), partitioners=("blocks", "equal_regions")):
    from paper_1908_07038_b200.partition import PARTITIONERS

    sg.set_device(0)
    g = sg.grid_from_name(grid)
    for pname in partitioners:
        for P in parts:
            dist = PARTITIONERS[pname](g, P)
            for h in halos:
                t0 = time.time()
                meshes = [sg.generate_mesh(g, dist, r, halo=h, include_pole=True) for r in range(P)]
                plans = sg.run_ranks(P, lambda ctx: sg.NodeColumns(meshes[ctx.rank], ctx).exchange_plan,
                                     devices=[0])
                fields = []
                for r, m in enumerate(meshes):
                    d = DeviceArray(m.nb_nodes, L, np.float64)
                    host = np.zeros((m.nb_nodes, L))
                    own = np.flatnonzero(~m.node_ghost)
                    host[own] = m.node_global[own, None] + np.arange(L)[None, :] * 1e-3
                    d.upload(host)
                    fields.append(d)
                info = [(d.ptr, d.pitch, d.device) for d in fields]
                pull_ms, pack_ms, ghosts, correct = [], [], [], True
                for r in range(P):
                    plan = plans[r]
                    nrecv = sum(len(v) for v in plan.recv.values())
                    nsend = sum(len(v) for v in plan.send.values())
                    ghosts.append(nrecv)
                    plan.pull(fields[r], info)
                    sg.synchronize(0)
                    got = fields[r].to_numpy()
                    m = meshes[r]
                    correct &= bool(np.array_equal(got, m.node_global[:, None] + np.arange(L)[None, :] * 1e-3))
                    e0, e1 = Event(0), Event(0)
                    e0.record()
                    for _ in range(REPS):
                        plan.pull(fields[r], info)
                    e1.record()
                    pull_ms.append(Event.elapsed_ms(e0, e1) / REPS)
                    buf = DeviceArray(1, max(nsend, nrecv, 1) * L, np.float64)
                    e0.record()
                    for _ in range(REPS):
                        plan.pack(fields[r], buf.ptr)
                        plan.unpack(fields[r], buf.ptr)
                    e1.record()
                    pack_ms.append(Event.elapsed_ms(e0, e1) / REPS)
                B = sum(ghosts) * L * 8
                worst = int(np.argmax(ghosts))
                print(json.dumps({
                    "grid": grid, "partitioner": pname, "levels": L, "parts": P, "halo": h, "ghosts_per_rank": ghosts,
                    "worst_rank": worst, "worst_rank_MB": ghosts[worst] * L * 8 / 1e6,
                    "bytes_per_exchange": B, "pull_ms_max": max(pull_ms), "pull_ms": pull_ms,
                    "pull_GBps_worst_rank": ghosts[worst] * L * 8 / (pull_ms[worst] * 1e-3) / 1e9,
                    "pack_unpack_ms_max": max(pack_ms), "values_correct": correct,
                    "note": "single-GPU emulation: peer memory is local HBM; per-rank kernels serialised",
                    "setup_s": round(time.time() - t0, 1)}), flush=True)
                for d in fields:
                    d.close()


if __name__ == "__main__":
    main()
