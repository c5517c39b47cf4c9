"""Small driver for profiling the stencil-search kernels: O1280 -> O640 serial locator build +
build_remap (tri boxes, bin fill, CUB sort, locate_kernel), then one in-process P=4 halo
exchange on O320 (pull kernel) and pack/unpack."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg
from paper_1908_07038_b200.device import DeviceArray

sg.set_device(0)
S, T = sg.grid_from_name("O1280"), sg.grid_from_name("O640")
dist = sg.blocks_partition(S, 1)
mesh = sg.generate_mesh(S, dist, 0, halo=2, include_pole=True)
w = sg.build_remap(sg.NodeColumns(mesh, None), T, sg.matching_partition(T, S, dist))
print("stencils", len(w))
g = sg.grid_from_name("O320")
d4 = sg.blocks_partition(g, 4)
meshes = [sg.generate_mesh(g, d4, r, halo=2, include_pole=True) for r in range(4)]
plans = sg.run_ranks(4, lambda ctx: sg.NodeColumns(meshes[ctx.rank], ctx).exchange_plan, devices=[0])
fields = [DeviceArray(m.nb_nodes, 137, np.float64) for m in meshes]
info = [(f.ptr, f.pitch, f.device) for f in fields]
for r in range(4):
    plans[r].pull(fields[r], info)
buf = DeviceArray(1, 200000 * 137, np.float64)
plans[1].pack(fields[1], buf.ptr)
plans[1].unpack(fields[1], buf.ptr)
sg.synchronize(0)
print("ok")
