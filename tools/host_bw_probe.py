"""Host memory bandwidth on the GPU box: numpy copies of a 4 GB buffer with 1/4/8/16 threads
(decides whether packing referenced rows on the host can beat PCIe for e2e)."""
import json, os, sys, time
from concurrent.futures import ThreadPoolExecutor
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1908_07038_b200.device import PinnedArray
n = 4 << 30
a = np.ones(n // 8)
b = PinnedArray((n // 8,)).array
b[:] = 0
out = {}
for T in (1, 4, 8, 16):
    chunks = np.array_split(np.arange(len(a)), T * 4)
    def job(i):
        s = slice(chunks[i][0], chunks[i][-1] + 1)
        b[s] = a[s]
    with ThreadPoolExecutor(T) as ex:
        list(ex.map(job, range(len(chunks))))
        t = time.perf_counter()
        list(ex.map(job, range(len(chunks))))
        dt = time.perf_counter() - t
    out[f"copy_GBps_{T}thr"] = n / dt / 1e9
print(json.dumps(out), flush=True)
del b
