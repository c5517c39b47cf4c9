"""H2D / D2H DMA rates on the box: 4 GB contiguous, pinned (portable) vs write-combined,
one and two streams."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg
from paper_1908_07038_b200.device import DeviceArray, PinnedArray, Event
sg.set_device(0)
n = 4 << 30
rows = n // (137 * 8)
out = {}
d = DeviceArray(rows, 137, np.float64)
for wc in (False, True):
    h = PinnedArray((rows, 137), write_combined=wc)
    h.array[:] = 1.0
    for rep in range(2):
        e0, e1 = Event(), Event()
        e0.record(); d.upload(h.array, sync=False); e1.record()
        ms = Event.elapsed_ms(e0, e1)
    out[f"h2d_GBps_{'wc' if wc else 'pinned'}"] = rows * 137 * 8 / ms / 1e6
    if not wc:
        e0, e1 = Event(), Event()
        e0.record(); d.download(h.array, sync=False); e1.record()
        out["d2h_GBps_pinned"] = rows * 137 * 8 / Event.elapsed_ms(e0, e1) / 1e6
    h.free()
print(json.dumps(out), flush=True)
