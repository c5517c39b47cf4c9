#!/usr/bin/env python
"""The REFERENCE's host halo_exchange (functionspace.py:107-118) at O1280, 137 levels, halo 2,
P=8 blocks (its own generate_mesh / NodeColumns / run_ranks), timed here for comparison with
tools/host_halo_timing.py.  Needs /root/reference (this container only); the meshes take
minutes in the reference's Python."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import spheregrid as R  # noqa: E402


def main():
    P, L = 8, 137
    S = R.grid_from_name("O1280")
    dist = R.blocks_partition(S, P)
    t_setup = time.perf_counter()

    def prog(ctx):
        mesh = R.generate_mesh(S, dist, ctx.rank, halo=2, include_pole=True)
        fs = R.NodeColumns(mesh, ctx)
        f = fs.create_field("src", L)
        own = ~mesh.node_ghost
        f.host[own] = mesh.node_global[own, None] * 1000.0 + np.arange(L)[None, :]
        fs.halo_exchange(f, ctx)
        ctx.barrier()
        t = time.perf_counter()
        for _ in range(3):
            fs.halo_exchange(f, ctx)
        ctx.barrier()
        dt = (time.perf_counter() - t) / 3
        ok = bool(np.array_equal(f.host, mesh.node_global[:, None] * 1000.0 + np.arange(L)[None, :]))
        ghosts = int(mesh.node_ghost.sum())
        return dt, ok, ghosts

    out = R.run_ranks(P, prog)
    ghosts = sum(o[2] for o in out)
    ms = max(o[0] for o in out) * 1e3
    print(json.dumps({"impl": "reference (numpy, run_ranks threads)", "grid": "O1280", "P": P, "levels": L, "halo": 2,
                      "partitioner": "blocks", "ms_per_exchange": round(ms, 2), "ghosts_total": ghosts,
                      "GB_per_exchange": ghosts * L * 8 / 1e9, "GB_per_s": ghosts * L * 8 / (ms * 1e-3) / 1e9,
                      "ghosts_equal_owners": all(o[1] for o in out),
                      "setup_s": round(time.perf_counter() - t_setup, 1), "host": "container CPU (8 cores)"}),
          flush=True)


if __name__ == "__main__":
    main()
