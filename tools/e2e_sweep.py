#!/usr/bin/env python
"""e2e sweep on cfg3 in one process: host-execute modes x gather CTAs/SM x pipeline chunks,
through the public apply_remap_fields on pinned host fields (bench.py's e2e leg).  One JSON
line per setting; every result checked bitwise against the first (dma) run."""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import paper_1908_07038_b200 as sg
    import paper_1908_07038_b200.interp as sgi
    from paper_1908_07038_b200.device import PinnedArray

    sg.set_device(0)
    S, T, mesh, fs, tdist, w = bench.setup_remap(sg, "O1280", "O640", 1, 0, None)
    m, n, L = len(w), mesh.nb_nodes, 137
    hsrc, hdst = PinnedArray((n, L)), PinnedArray((m, L))
    bench.fill_smooth(hsrc.array, mesh.node_xyz, 0)
    if os.environ.get("CREATE") == "1":  # host mirrors from the public create_field
        t = time.perf_counter()
        a = sg.create_field("src", (n, L))
        print(json.dumps({"create_field_s": round(time.perf_counter() - t, 3), "pinned": sgi._is_pinned(a.host)}),
              flush=True)
        a.host[:] = hsrc.array
        fsrc, fdst = a, sg.create_field("dst", (m, L))
        hsrc, hdst = None, None
    elif os.environ.get("PAGEABLE") == "1":  # plain numpy arrays (user-supplied host storage)
        class _A:
            pass
        a, b = _A(), _A()
        a.array, b.array = hsrc.array.copy(), np.zeros((m, L))
        hsrc, hdst = a, b
    if hsrc is not None:
        fsrc = sg.Field(name="src", shape=(n, L), kind=sg.Kind.REAL64, host=hsrc.array)
        fdst = sg.Field(name="dst", shape=(m, L), kind=sg.Kind.REAL64, host=hdst.array)
    ref = None
    settings = [("dma", 2, 64)]
    env = os.environ.get("SWEEP_ENV", "SG_GATHER_CTAS")  # knob swept in the third column
    vals = [int(x) for x in os.environ.get("SWEEP_VALS", "2,4,8").split(",")]
    chunks = [int(x) for x in os.environ.get("SWEEP_CHUNKS", "32,64,128").split(",")]
    for mode in sys.argv[1].split(",") if len(sys.argv) > 1 else ["gather"]:
        for v in vals:
            for ch in chunks:
                settings.append((mode, v, ch))
    for mode, ctas, ch in settings:
        os.environ[env] = str(ctas)
        sgi.HOST_EXECUTE_MODE, sgi.HOST_EXECUTE_CHUNKS = mode, ch
        fdst.host[:] = 0
        for _ in range(3):
            sg.apply_remap_fields(w, [fsrc], [fdst])
        ts = []
        for _ in range(8):
            t = time.perf_counter()
            sg.apply_remap_fields(w, [fsrc], [fdst])
            ts.append(time.perf_counter() - t)
        if ref is None:
            ref = fdst.host.copy()
        ok = bool(np.array_equal(ref.view(np.uint64), fdst.host.view(np.uint64)))
        ms = statistics.median(ts) * 1e3
        print(json.dumps({"mode": mode, env: ctas, "chunks": ch, "ms": round(ms, 2),
                          "gpts_lev_s": round(m * L / (ms * 1e-3) / 1e9, 4), "bitwise": ok}), flush=True)


if __name__ == "__main__":
    main()
