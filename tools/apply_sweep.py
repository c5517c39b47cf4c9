"""Apply-kernel variant sweep on cfg3 (O1280 -> O640, 137 levels): per variant the mean
kernel time over 20 launches, two interleaved rounds.  Variants: 0 default (8-B loads),
2/6/7 TMA bulk tiles, 4/5 L2 prefetch hints (apply.cu launch_apply).  Experimental
variants measured once and removed are listed in profiles/r01_apply_variant_sweep2.jsonl.
Usage: apply_sweep.py [comma-separated variants]"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg
from paper_1908_07038_b200.device import DeviceArray, Event
from oracle import oracle as O

sg.set_device(0)
S, T = sg.grid_from_name("O1280"), sg.grid_from_name("O640")
dist = sg.blocks_partition(S, 1)
mesh = sg.generate_mesh(S, dist, 0, halo=2, include_pole=True)
w = sg.build_remap(sg.NodeColumns(mesh, None), T, sg.matching_partition(T, S, dist))
L = 137
host = np.random.default_rng(0).normal(size=(mesh.nb_nodes, L))
src, dst = DeviceArray(mesh.nb_nodes, L, np.float64), DeviceArray(len(w), L, np.float64)
src.upload(host)
B = 7342176168
samp = np.random.default_rng(1).choice(len(w), 3000, replace=False)
exp = O.apply_remap(w.nodes[samp], w.weights[samp], host)
res = {}
for rnd in range(2):
    for v in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['0', '2', '6', '7'])]:
        for _ in range(3):
            sg.apply_remap_device(w, [src], [dst], variant=v)
        e0, e1 = Event(), Event()
        e0.record()
        for _ in range(20):
            sg.apply_remap_device(w, [src], [dst], variant=v)
        e1.record()
        ms = Event.elapsed_ms(e0, e1) / 20
        ok = bool(np.array_equal(dst.to_numpy()[samp].view(np.uint64), exp.view(np.uint64)))
        res.setdefault(v, []).append(ms)
        print(json.dumps({"variant": v, "round": rnd, "ms": ms, "GBps_alg": B / ms / 1e6,
                          "frac": B / ms / 1e6 / 6535.4, "bitwise": ok}), flush=True)
