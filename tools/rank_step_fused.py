#!/usr/bin/env python
"""Per-rank N>1 step time measured on ONE GPU: the cfg3 decomposition (O1280 -> O640, 137
lev, halo 2) at P = 2 / 4 / 8, every rank's FUSED signalled step (signal kernel + step kernel
with PDL, csrc/step.cu) launched ALONE on its own data with its owners' ready words
pre-published (Signal.publish_owners_ahead), CUDA events, mean of 20.  The max over ranks is
one GPU's share of a P-GPU step minus NVLink latency of the ~0.1 % boundary rows (peer rows
come from this GPU's HBM here); efficiency = (N=1 apply time / P) / max over ranks.  Beside it,
each rank's plain apply launch over the same data (ghost rows local, no signalling).
Prints one JSON line per (partitioner, P); used for profiles/r02_rank_step_fused_1gpu.jsonl."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_07038_b200 as sg  # noqa: E402
from paper_1908_07038_b200.device import DeviceArray, Event, Stream  # noqa: E402
from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps  # noqa: E402
from paper_1908_07038_b200.partition import PARTITIONERS  # noqa: E402

sg.set_device(0)
S, T = sg.grid_from_name("O1280"), sg.grid_from_name("O640")
L, REPS = 137, 20
st = Stream(0)


def time_it(fn):
    for _ in range(3):
        fn()
    e0, e1 = Event(0), Event(0)
    e0.record(st.stream)
    for _ in range(REPS):
        fn()
    e1.record(st.stream)
    st.synchronize()
    return Event.elapsed_ms(e0, e1) / REPS


# N = 1: the plain apply of the whole configuration (skipped with NO_SERIAL=1)
t1 = 1.0852  # profiles/r02_rank_step_fused_1gpu.jsonl
if not os.environ.get("NO_SERIAL"):
    dist1 = sg.blocks_partition(S, 1)
    mesh1 = sg.generate_mesh(S, dist1, 0, halo=2, include_pole=True)
    w1 = sg.build_remap(sg.NodeColumns(mesh1, None), T, sg.matching_partition(T, S, dist1))
    a1, b1 = DeviceArray(mesh1.nb_nodes, L, np.float64), DeviceArray(len(w1), L, np.float64)
    t1 = time_it(lambda: sg.apply_remap_device(w1, [a1], [b1], stream=st.stream))
    del a1, b1
    print(json.dumps({"P": 1, "apply_ms": t1}), flush=True)

PARTS = [int(x) for x in os.environ.get("PARTS", "2,4,8").split(",")]
PARTITIONERS_RUN = os.environ.get("PARTITIONERS", "equal_regions,blocks").split(",")
for pname in PARTITIONERS_RUN:
    for P in PARTS:
        dist = PARTITIONERS[pname](S, P)
        td = sg.matching_partition(T, S, dist)

        def prog(ctx):
            mesh = sg.generate_mesh(S, dist, ctx.rank, halo=2, include_pole=True)
            fs = sg.NodeColumns(mesh, ctx)
            w = sg.build_remap(fs, T, td, ctx)
            src = DeviceArray(mesh.nb_nodes, L, np.float64)
            src.upload(np.random.default_rng(ctx.rank).normal(size=(mesh.nb_nodes, L)))
            return w, fs.exchange_plan, src, DeviceArray(len(w), L, np.float64)

        ranks = sg.run_ranks(P, prog, devices=[0])
        steps = emulated_fused_steps(ranks)
        per, plain = [], []
        for r, s in enumerate(steps):
            s.signal.publish_owners_ahead(1 << 40)
            per.append(time_it(lambda s=s: launch_fused_steps([s], st.stream)))
            s.check()
            w, _, src, dst = ranks[r]
            plain.append(time_it(lambda: sg.apply_remap_device(w, [src], [dst], stream=st.stream)))
        worst = max(per)
        print(json.dumps({"partitioner": pname, "P": P, "per_rank_step_ms": [round(x, 4) for x in per],
                          "per_rank_plain_apply_ms": [round(x, 4) for x in plain],
                          "worst_ms": worst, "worst_plain_apply_ms": max(plain), "ideal_ms": t1 / P,
                          "compute_efficiency": t1 / P / worst,
                          "targets": [s.m for s in steps], "boundary_targets": [s.n_boundary for s in steps]}),
              flush=True)
        del ranks, steps
