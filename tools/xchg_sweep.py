#!/usr/bin/env python
"""cfg4 point (O1280, 137 lev, halo H, equal regions P ranks) emulated on one GPU: all ranks'
signalled pulls (sg_exchange_*) as one launch.  Prints one JSON line (median of 10; before
every launch the L2 is flushed by a 2 GiB read (FLUSH=read) or a 512 MB copy (FLUSH=copy, the
default measurement of profiles/r02_exchange_signalled.md: dirty L2 as after a source update))."""
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_07038_b200 as sg  # noqa: E402
from paper_1908_07038_b200.device import DeviceArray, Event  # noqa: E402
from paper_1908_07038_b200.execute import emulated_exchanges, launch_exchanges  # noqa: E402
from paper_1908_07038_b200.partition import PARTITIONERS  # noqa: E402

P, H, L = int(os.environ.get("PARTS", 8)), int(os.environ.get("HALO", 2)), int(os.environ.get("LEVELS", 137))
S = sg.grid_from_name(os.environ.get("GRID", "O1280"))
dist = PARTITIONERS[os.environ.get("PART", "equal_regions")](S, P)
meshes = [sg.generate_mesh(S, dist, r, halo=H, include_pole=True) for r in range(P)]
plans = sg.run_ranks(P, lambda ctx: sg.NodeColumns(meshes[ctx.rank], ctx).exchange_plan, devices=[0])
fields = []
for m in meshes:
    d = DeviceArray(m.nb_nodes, L, np.float64)
    vals = m.node_global[:, None].astype(np.float64) + np.arange(L)[None, :] / L
    d.upload(np.where(m.node_ghost[:, None], -1.0, vals))
    fields.append(d)
flush = DeviceArray(1 << 22, 64, np.float64)  # 2 GiB > L2
gid0 = np.zeros(1 << 22, np.int64)
part = C.c_uint64(0)
xs = emulated_exchanges(list(zip(plans, fields)))
launch_exchanges(xs)
ok = all(np.array_equal(f.to_numpy(), m.node_global[:, None].astype(np.float64) + np.arange(L)[None, :] / L)
         for f, m in zip(fields, meshes))
t = []
for _ in range(10):
    mode = os.environ.get("FLUSH", "copy")
    if mode == "read":  # read 2 GiB: evicts L2 with clean lines
        sg._native.call("sg_field_checksum", flush.handle, 0, 1 << 22, gid0.ctypes.data, C.byref(part))
    elif mode == "copy":  # copy 512 MB: leaves L2 full of dirty lines, written back during the timed launch
        sg._native.call("sg_rows_copy", 0, flush.ptr, 512, 0, flush.ptr + 256, 512, 0, 1 << 21, 256, 0)
    # "none": back-to-back exchanges, warm L2 (the steady state of repeated exchanges)
    e0, e1 = Event(0), Event(0)
    e0.record()
    launch_exchanges(xs)
    e1.record()
    t.append(Event.elapsed_ms(e0, e1))
nb = sum(sum(len(v) for v in p.recv.values()) for p in plans) * L * 8
ms = statistics.median(t)
print(json.dumps({"P": P, "halo": H, "levels": L, "flush": os.environ.get("FLUSH", "copy"),

                  "bytes": nb, "ms": ms, "GB_per_s": nb / (ms * 1e-3) / 1e9, "ghosts_bitwise": ok,
                  "epochs": [x.check() for x in xs]}))
