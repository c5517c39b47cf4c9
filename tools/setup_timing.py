"""Host-side setup, timed in this container: the reference's Python
(gaussian_latitudes, generate_mesh, matching_partition) against the native/vectorised
drop-in, on the same host, with bit-identical results checked.  Needs /root/reference (run
here, not on the GPU box).  Prints one JSON line per (function, size)."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import spheregrid as R
import paper_1908_07038_b200 as M


def timed(fn, *a, **k):
    t = time.perf_counter()
    out = fn(*a, **k)
    return out, time.perf_counter() - t


for n in (160, 320, 640):
    ref, tr = timed(R.gaussian_latitudes, n)
    mine, tm = timed(M.gaussian_latitudes, n)
    print(json.dumps({"fn": "gaussian_latitudes", "n": n, "reference_s": tr, "b200_pkg_s": tm,
                      "bitwise": bool(np.array_equal(ref.view(np.uint64), mine.view(np.uint64)))}), flush=True)
for name, P, h in (("O160", 1, 2), ("O320", 1, 2), ("O320", 8, 2)):
    gr, gm = R.grid_from_name(name), M.grid_from_name(name)
    dr, dm = R.blocks_partition(gr, P), M.blocks_partition(gm, P)
    r = P // 2
    a, tr = timed(R.generate_mesh, gr, dr, r, halo=h, include_pole=True)
    b, tm = timed(M.generate_mesh, gm, dm, r, halo=h, include_pole=True)
    same = all(np.array_equal(getattr(a, k), getattr(b, k)) for k in
               ("node_global", "node_xyz", "node_part", "node_remote", "node_halo", "elem_serial_id"))
    same &= np.array_equal(a.element_connectivity.indices, b.element_connectivity.indices)
    print(json.dumps({"fn": "generate_mesh", "grid": name, "parts": P, "rank": r, "halo": h, "reference_s": tr,
                      "b200_pkg_s": tm, "bitwise": bool(same)}), flush=True)
for tgt, src, P in (("O80", "O160", 8), ("O160", "O320", 8)):
    S, T = R.grid_from_name(src), R.grid_from_name(tgt)
    a, tr = timed(R.matching_partition, T, S, R.blocks_partition(S, P))
    Sm, Tm = M.grid_from_name(src), M.grid_from_name(tgt)
    b, tm = timed(M.matching_partition, Tm, Sm, M.blocks_partition(Sm, P))
    print(json.dumps({"fn": "matching_partition", "target": tgt, "source": src, "parts": P, "reference_s": tr,
                      "b200_pkg_s": tm, "bitwise": bool(np.array_equal(a.part_of, b.part_of))}), flush=True)
