#!/usr/bin/env python
"""The fused distributed step (csrc/step.cu) of cfg3 at P ranks EMULATED on one GPU as one
launch over every rank's data (bench.py emulated_fused_step), run on its own so that ncu can
capture step_kernel:  ncu -k regex:step_kernel -s 3 -c 1 python tools/fused_step_emulated.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_07038_b200 as sg  # noqa: E402

P = int(os.environ.get("PARTS", "8"))
r = bench.emulated_fused_step(sg, "O1280", "O640", 137, parts=P, reps=int(os.environ.get("REPS", "10")))
print(json.dumps({k: v for k, v in r.items() if k != "scope"}))
