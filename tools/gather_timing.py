#!/usr/bin/env python
"""gather_field / scatter_field at O1280 x 137 levels fp64 (the cfg3 source), P = 1 and P = 4
in-process ranks on one GPU: the device path (sg_rows_copy from each rank's HBM + one D2H;
one H2D + per-rank pulls for scatter) against the reference algorithm on the host
(functionspace.py:185-224, numpy fancy indexing; `_gather_host` / `_scatter_host`).  Prints
one JSON line per case; used for profiles/r02_gather_scatter_o1280.jsonl."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_07038_b200 as sg  # noqa: E402
import paper_1908_07038_b200.functionspace as FS  # noqa: E402

L = 137
g = sg.grid_from_name(os.environ.get("GRID", "O1280"))
gvals = np.random.default_rng(3).normal(size=(g.npts + 2, L))


def case(P, device_dirty):
    def program(ctx):
        c = ctx if ctx.nranks > 1 else None
        dist = sg.blocks_partition(g, ctx.nranks)
        mesh = sg.generate_mesh(g, dist, ctx.rank, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, c)
        f = fs.create_field("x", L)
        own = fs.owned_row_index()
        f.host[own] = gvals[mesh.node_global[own]]
        if device_dirty:
            f.allocate_device()
            with f.device_view(sg.Intent.READ_WRITE):
                pass
        out = {}
        for name, fn in (("device", sg.gather_field), ("host_reference_algorithm", FS._gather_host)):
            ts = []
            for _ in range(3):
                if c is not None:
                    ctx.barrier()
                t = time.perf_counter()
                res = fn(fs, f, c)
                if c is not None:
                    ctx.barrier()
                ts.append(time.perf_counter() - t)
            out[f"gather_{name}_s"] = min(ts)
            if ctx.rank == 0:
                out[f"gather_{name}_ok"] = bool(np.array_equal(res, gvals))
        sfs = sg.StructuredColumns(g, dist, ctx.rank)
        sf = sfs.create_field("s", L)
        for name, fn in (("device", sg.scatter_field), ("host_reference_algorithm", FS._scatter_host)):
            ts = []
            for _ in range(3):
                if c is not None:
                    ctx.barrier()
                t = time.perf_counter()
                fn(sfs, sf, c, gvals[: g.npts] if ctx.rank == 0 else None)
                if c is not None:
                    ctx.barrier()
                ts.append(time.perf_counter() - t)
            out[f"scatter_{name}_s"] = min(ts)
            out[f"scatter_{name}_ok"] = bool(np.array_equal(sf.host, gvals[sfs.owned_global]))
        return out

    r = sg.run_ranks(P, program, devices=[0])
    line = {"grid": g.name, "levels": L, "P": P, "field_state": "DEVICE_DIRTY" if device_dirty else "HOST_ONLY",
            "global_bytes": int((g.npts + 2) * L * 8), **r[0],
            "scatter_ok_all_ranks": all(x["scatter_device_ok"] for x in r)}
    print(json.dumps(line), flush=True)


for P in (1, 4):
    for dd in (False, True):
        case(P, dd)
