"""Probe: CUDA-IPC handles of small per-object allocations (step signal words).  Rank 0 makes
three Signals and a field, writes distinct words, shares the IPC handles; rank 1 opens each,
reads the words through the mapped pointer (sg_rows_copy into its own buffer), then closes
mapping 0 and reads mapping 1 again.  Prints one JSON line from rank 1."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main(rank, q_in, q_out):
    import ctypes as C

    import paper_1908_07038_b200 as sg
    from paper_1908_07038_b200 import _native as N
    from paper_1908_07038_b200.device import DeviceArray
    from paper_1908_07038_b200.execute import Signal

    sg.set_device(0)
    if rank == 0:
        sigs = [Signal(0, 2, 0) for _ in range(3)]
        out = []
        for k, s in enumerate(sigs):
            w = np.arange(8, dtype=np.uint64) + 1000 * (k + 1)
            N.call("sg_signal_write", s.handle, N.ptr(w), len(w))
            h = (C.c_uint8 * 64)()
            N.call("sg_signal_ipc_handle", s.handle, N.ref(h), 64)
            out.append((bytes(h).hex(), s.ptr))
        q_out.put(out)
        q_in.get()  # keep alive until rank 1 is done
        return
    handles = q_in.get()
    res = {"same_handle_01": handles[0][0] == handles[1][0], "same_handle_12": handles[1][0] == handles[2][0],
           "ptr_deltas": [handles[k][1] - handles[0][1] for k in range(3)]}
    buf = DeviceArray(1, 8, np.uint64)
    ptrs = []
    for k, (hx, _) in enumerate(handles):
        h = (C.c_uint8 * 64).from_buffer_copy(bytes.fromhex(hx))
        p = C.c_uint64(0)
        try:
            N.call("sg_ipc_open", 0, N.ref(h), 64, N.ref(p))
        except Exception as e:  # noqa: BLE001
            res[f"open_{k}"] = repr(e)[:200]
            ptrs.append(None)
            continue
        ptrs.append(p.value)
        N.call("sg_rows_copy", 0, buf.ptr, 64, 0, p.value, 64, 0, 1, 64, 0)
        res[f"words_{k}"] = buf.to_numpy().ravel()[:2].tolist()
    res["opened_ptr_deltas"] = [(x - ptrs[0]) if (x is not None and ptrs[0] is not None) else None for x in ptrs]
    if ptrs[0] is not None:
        N.call("sg_ipc_close", 0, ptrs[0])
        try:
            N.call("sg_rows_copy", 0, buf.ptr, 64, 0, ptrs[1], 64, 0, 1, 64, 0)
            res["words_1_after_close_0"] = buf.to_numpy().ravel()[:2].tolist()
        except Exception as e:  # noqa: BLE001
            res["words_1_after_close_0"] = repr(e)[:200]
        try:
            N.call("sg_rows_copy", 0, buf.ptr, 64, 0, ptrs[0], 64, 0, 1, 64, 0)
            res["words_0_after_close_0"] = buf.to_numpy().ravel()[:2].tolist()
        except Exception as e:  # noqa: BLE001
            res["words_0_after_close_0"] = repr(e)[:200]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    a, b = ctx.Queue(), ctx.Queue()
    p0 = ctx.Process(target=main, args=(0, b, a))
    p0.start()
    handles = a.get()
    p1 = ctx.Process(target=main, args=(1, None, None))
    # rank 1 reads the handles from its own queue
    q = ctx.Queue()
    q.put(handles)
    p1 = ctx.Process(target=main, args=(1, q, None))
    p1.start()
    p1.join(120)
    b.put(1)
    p0.join(60)
