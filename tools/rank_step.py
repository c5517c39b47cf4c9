"""Per-rank compute of the cfg3 decomposition, measured on ONE GPU: for P in 1/2/4/8
(blocks and equal regions), the worst rank's apply (its targets, its local mesh with halo
2) timed with CUDA events, plus the same step captured as a CUDA graph with the interior /
boundary target lists.  Compute-only strong-scaling evidence: the cross-GPU exchange needs
more than one GPU."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_07038_b200 as sg
from paper_1908_07038_b200.device import DeviceArray, Event
from paper_1908_07038_b200.execute import DistributedRemap
from paper_1908_07038_b200.partition import PARTITIONERS

sg.set_device(0)
S, T = sg.grid_from_name("O1280"), sg.grid_from_name("O640")
L = 137
base_ms = None
for pname in ("blocks", "equal_regions"):
    for P in (1, 2, 4, 8):
        dist = PARTITIONERS[pname](S, P)
        td = sg.matching_partition(T, S, dist)
        counts = np.bincount(td.part_of, minlength=P)
        r = int(np.argmax(counts))
        mesh = sg.generate_mesh(S, dist, r, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, None)
        w = sg.build_remap(fs, T, td)
        src = DeviceArray(mesh.nb_nodes, L, np.float64)
        src.upload(np.random.default_rng(r).normal(size=(mesh.nb_nodes, L)))
        dst = DeviceArray(len(w), L, np.float64)
        for _ in range(3):
            sg.apply_remap_device(w, [src], [dst])
        e0, e1 = Event(), Event()
        e0.record()
        for _ in range(20):
            sg.apply_remap_device(w, [src], [dst])
        e1.record()
        ms = Event.elapsed_ms(e0, e1) / 20
        run = DistributedRemap(fs, w, None, src, dst)
        run.step(); run.synchronize(); run.capture()
        for _ in range(3):
            run.step()
        g0, g1 = Event(), Event()
        g0.record(run.main.stream)
        for _ in range(20):
            run.step()
        g1.record(run.main.stream)
        gms = Event.elapsed_ms(g0, g1) / 20
        if P == 1 and pname == "blocks":
            base_ms = ms
        U = w.distinct_sources()
        B = U * L * 8 + len(w) * L * 8 + len(w) * 36
        print(json.dumps({"partitioner": pname, "parts": P, "worst_rank": r, "targets": len(w),
                          "nodes": mesh.nb_nodes, "apply_ms": ms, "graph_step_ms": gms,
                          "frac_of_peak": B / ms / 1e6 / 6535.4,
                          "compute_scaling_eff": base_ms / (P * ms) if base_ms else None}), flush=True)
