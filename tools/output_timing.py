"""§8(f) row 2 timing: device checksum / gather of an O1280 x 137 field vs the reference
algorithm's numpy restatement (oracle.checksum_partial, single thread) on the box host."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg
from oracle import oracle as O

sg.set_device(0)
for name in ("O640", "O1280"):
    g = sg.grid_from_name(name)
    fs = sg.StructuredColumns(g, sg.blocks_partition(g, 1), 0)
    f = fs.create_field("v", 137)
    f.host[:] = np.random.default_rng(1).normal(size=f.host.shape)
    f.allocate_device()
    sg.checksum(fs, f, None)  # warm
    t = time.perf_counter()
    d = sg.checksum(fs, f, None)
    gpu_s = time.perf_counter() - t
    t = time.perf_counter()
    ref = O.checksum_partial(fs.owned_global, f.host)
    cpu_s = time.perf_counter() - t
    n = f.npts * f.levels
    print(json.dumps({"grid": name, "levels": 137, "values": n, "checksum_equal": d == ref,
                      "device_checksum_s": gpu_s, "device_Gvalues_per_s": n / gpu_s / 1e9,
                      "reference_numpy_s": cpu_s, "reference_Gvalues_per_s": n / cpu_s / 1e9,
                      "note": "device time includes the gid upload and the host round trip of one call"}), flush=True)
