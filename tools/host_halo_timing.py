#!/usr/bin/env python
"""Host-field NodeColumns.halo_exchange (functionspace.py:107-118 semantics) on in-process
ranks sharing one GPU: O1280, 137 levels, halo 2, P=8, blocks and equal regions.  Times the
exchange as shipped (only the rows peers read are staged on the device) against staging the
whole field (the previous implementation), and checks ghosts == owners' values."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1908_07038_b200 as sg
    from paper_1908_07038_b200.functionspace import _staging
    from paper_1908_07038_b200.partition import PARTITIONERS

    S, L, P = sg.grid_from_name("O1280"), 137, 8
    for part in ("blocks", "equal_regions"):
        dist = PARTITIONERS[part](S, P)

        def prog(ctx):
            mesh = sg.generate_mesh(S, dist, ctx.rank, halo=2, include_pole=True)
            fs = sg.NodeColumns(mesh, ctx)
            f = fs.create_field("src", L)
            own = fs.owned_row_index()
            f.host[own] = (mesh.node_global[own, None] * 1000 + np.arange(L)[None, :]).astype(np.float64)
            fs.halo_exchange(f, ctx)  # warm: staging buffer, plan upload
            ctx.barrier()
            t = time.perf_counter()
            for _ in range(5):
                fs.halo_exchange(f, ctx)
            ctx.barrier()
            new_s = (time.perf_counter() - t) / 5
            ok = bool(np.array_equal(f.host, (mesh.node_global[:, None] * 1000 + np.arange(L)[None, :]).astype(np.float64)))
            plan = fs.exchange_plan
            ctx.barrier()
            t = time.perf_counter()
            for _ in range(5):  # previous implementation: whole field staged
                dev = _staging(f)
                dev.upload(f.host)
                ctx.device_exchange(plan, dev)
                lo, hi = plan.ghost_rows
                f.host[lo:hi] = dev.download_rows(lo, hi - lo)
            ctx.barrier()
            old_s = (time.perf_counter() - t) / 5
            ghosts = sum(len(v) for v in plan.recv.values())
            return new_s, old_s, ok, int(plan.send_runs().shape[0]), ghosts, mesh.nb_nodes

        out = sg.run_ranks(P, prog, devices=[0])
        print(json.dumps({"partitioner": part, "P": P, "levels": L,
                          "ms_per_exchange_staged_send_rows": round(max(o[0] for o in out) * 1e3, 2),
                          "ms_per_exchange_staged_whole_field": round(max(o[1] for o in out) * 1e3, 2),
                          "ghosts_total": sum(o[4] for o in out), "send_runs_max": max(o[3] for o in out),
                          "nodes_per_rank_max": max(o[5] for o in out), "ghosts_equal_owners": all(o[2] for o in out)}),
              flush=True)


if __name__ == "__main__":
    main()
