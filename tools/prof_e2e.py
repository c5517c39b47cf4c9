#!/usr/bin/env python
"""One cfg3 e2e call (apply_remap_fields on pinned host fields, gather mode) for ncu: the
launch list shows the pipeline's kernels (gather_tma chunks pulling referenced rows over PCIe,
apply chunks from the compact device copy).  Not a timing run."""
import os
import sys

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
    hsrc.array[:] = np.random.default_rng(0).normal(size=(n, L))
    fsrc = sg.Field(name="src", shape=(n, L), kind=sg.Kind.REAL64, host=hsrc.array)
    fdst = sg.Field(name="dst", shape=(m, L), kind=sg.Kind.REAL64, host=hdst.array)
    sgi.HOST_EXECUTE_MODE = "gather"
    for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
        sg.apply_remap_fields(w, [fsrc], [fdst])
    print("rows moved", w.last_host_rows_moved, "of", n)


if __name__ == "__main__":
    main()
