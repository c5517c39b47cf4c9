#!/usr/bin/env python
"""Wall time of the whole reference pipeline (run_remap_pipeline, cli.py:119-154) on the
device path: O1280 -> O640, 1 level, P in-process ranks sharing GPU 0 — grid, latitudes,
partition, per-rank mesh (halo 2), matching partition, halo exchange, build_remap, apply,
gather to rank 0.  Reference: ~2.5 h at P=1 by the survey's per-stage measurements
(latitudes 45 s + xyz 55 s + mesh 120 s + matching 24 s + locator 69 s + build ~1.9 h)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1908_07038_b200 as sg

    for P in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8").split(",")]:
        for part in ("blocks", "equal_regions"):
            t = time.perf_counter()
            got, exact, msgs = sg.run_remap_pipeline("O1280", "O640", P, "harmonic:Y3,1", devices=[0], partitioner=part)
            wall = time.perf_counter() - t
            err = np.abs(got - exact)
            print(json.dumps({"P": P, "partitioner": part, "wall_s": round(wall, 2), "max_error": float(err.max()),
                              "messages_during_interpolation": int(sum(msgs))}), flush=True)


if __name__ == "__main__":
    main()
