"""Stencil parity at the largest scale: O2560 -> O1280 finite-element remap (26.3 M source
nodes, 52.6 M triangles, 6.6 M targets).  The device build is compared with the scaled
oracle (the reference algorithm: scipy cKDTree k=8/32 candidates + its scoring) on every
target; timings of both are reported."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg
from oracle import oracle as O

sg.set_device(0)
S, T = sg.grid_from_name("O2560"), sg.grid_from_name("O1280")
t0 = time.perf_counter()
dist = sg.blocks_partition(S, 1)
mesh = sg.generate_mesh(S, dist, 0, halo=2, include_pole=True)
t_mesh = time.perf_counter() - t0
t0 = time.perf_counter()
loc = sg.MeshLocator(mesh)
t_loc = time.perf_counter() - t0
t0 = time.perf_counter()
w = sg.build_remap(sg.NodeColumns(mesh, None), T, sg.matching_partition(T, S, dist), locator=loc)
t_build = time.perf_counter() - t0
conn = mesh.element_connectivity
txyz = T.xyz()
t0 = time.perf_counter()
e, c = O.locate_kdtree(mesh.node_xyz, conn.offsets, conn.indices, txyz)
t_oracle = time.perf_counter() - t0
ow = O.barycentric_weights_batched(mesh.node_xyz, c, txyz)
print(json.dumps({"source": "O2560", "target": "O1280", "source_nodes": mesh.nb_nodes, "targets": len(w),
                  "locator": loc.stats(), "mesh_s": t_mesh, "locator_s": t_loc, "build_remap_s": t_build,
                  "oracle_locate_s": t_oracle, "oracle_unlocated": int((e < 0).sum()),
                  "stencil_mismatches": int((w.nodes != c).any(axis=1).sum()),
                  "max_weight_diff": float(np.abs(w.weights - ow).max()),
                  "weights_bitwise": bool(np.array_equal(w.weights.view(np.uint64), ow.view(np.uint64)))}), flush=True)
