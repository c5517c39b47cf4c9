#!/usr/bin/env python
"""First vs later calls of apply_remap on host fields at cfg3 (gather mode, pinned mirrors):
the first call also builds the stencil's host plan (profiles/r01_e2e_modes.md)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import paper_1908_07038_b200 as sg
    from paper_1908_07038_b200.device import PinnedArray

    sg.set_device(0)
    S, T, mesh, fs, tdist, w = bench.setup_remap(sg, "O1280", "O640", 1, 0, None)
    m, n, L = len(w), mesh.nb_nodes, 137
    hs, hd = PinnedArray((n, L)), PinnedArray((m, L))
    hs.array[:] = 1.0
    f = sg.Field(name="s", shape=(n, L), kind=sg.Kind.REAL64, host=hs.array)
    g = sg.Field(name="d", shape=(m, L), kind=sg.Kind.REAL64, host=hd.array)
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        sg.apply_remap(w, f, g)
        ts.append(round((time.perf_counter() - t) * 1e3, 1))
    print(json.dumps({"config": "cfg3 host fields, gather mode", "call_ms": ts}), flush=True)


if __name__ == "__main__":
    main()
