"""First and steady-state calls of apply_remap on host fields at cfg3 (O1280 -> O640, 137 lev):
the first call builds the gather plan (on the device since round 2).  Prints ms per call."""
import os, sys, time, numpy as np
sys.path.insert(0, os.getcwd())
import bench, paper_1908_07038_b200 as sg
from paper_1908_07038_b200.device import PinnedArray
S, T, mesh, fs, tdist, w = bench.setup_remap(sg, "O1280", "O640", 1, 0, None)
n, m, L = mesh.nb_nodes, len(w), 137
hs = PinnedArray((n, L)); hd = PinnedArray((m, L)); hs.array[:] = 1.0
fs_ = sg.Field(name="s", shape=(n, L), kind=sg.Kind.REAL64, host=hs.array)
fd = sg.Field(name="d", shape=(m, L), kind=sg.Kind.REAL64, host=hd.array)
for k in range(4):
    t = time.perf_counter(); sg.apply_remap_fields(w, [fs_], [fd]); print("call", k, round((time.perf_counter() - t) * 1e3, 1), "ms", flush=True)
