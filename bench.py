#!/usr/bin/env python
"""Benchmark of the hot path: O1280 -> O640 linear finite-element remap of a 137-level fp64
field (BASELINE.json configs[2], the metric's configuration; it fits one B200).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one execute of the remap over the whole configuration: at N=1 the apply kernel
(interp.py:206-228 on the device); at N>1 (torchrun, one process per GPU, blocks_partition
+ matching_partition, mesh halo 2) the NodeColumns halo exchange of the source field (pack ->
NCCL send/recv -> unpack) followed by the apply.  ``value`` is whole-job Gpts·lev/s with the
inputs resident in HBM; ``e2e`` is the same metric through the public API
(``apply_remap`` on host-resident fields in pinned memory: h2d of the source field, the
kernel, d2h of the target field, every step).  Inputs (7.3 GB) exceed the 126 MB L2, so no
flush is needed between steps.  ``--impl reference`` times the reference's CPU apply (the
oracle port of interp.py:219-223, numpy, all host threads) on the same configuration.
Synthetic data: level k of the field = Y_{l,m}(xyz)·(1 + k/L), (l, m) cycling through the 25
real harmonics l <= 4.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (source, target, levels, fields[, method])
    "cfg3": ("O1280", "O640", 137, 1),
    "cfg2": ("O320", "O160", 137, 4),
    "cfg1": ("O32", "O16", 10, 1),
    # structured bilinear: no reference method (parity vs oracle.bilinear_stencil only)
    "cfg5": ("O2560", "O1280", 137, 1, "bilinear"),
    # the finite-element method at cfg5's size (stencils bit-exact vs the scaled oracle,
    # profiles/r01_scale_parity_o2560.json)
    "cfg5fe": ("O2560", "O1280", 137, 1),
}


def metric_name(source, target, method, L):
    if (source, target, method, L) == ("O1280", "O640", "fe", 137):
        return METRIC
    kind = "structured-bilinear" if method == "bilinear" else "FE"
    return f"Gpts·lev/s {source}→{target} {kind} interp, {L} lev fp64"


def config(name):
    c = CONFIGS[name]
    return c[0], c[1], c[2], c[3], (c[4] if len(c) > 4 else "fe")
def _baseline_metric() -> str:
    """BASELINE.json's metric string verbatim (the roofline fraction and the halo GB/s it
    names are the line's ``roofline.frac`` and, at N>1, ``halo.GB_per_s``)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as fh:
            return json.load(fh)["metric"]
    except (OSError, KeyError, ValueError):
        return "Gpts·lev/s O1280→O640 FE interp, 137 lev fp64; % HBM roofline; halo GB/s"


METRIC = _baseline_metric()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config: str):
    """dram bytes per launch of the apply kernel from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_apply_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(config, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed regions."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.active = False
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            if self.active:
                self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


HARMONICS = [(l, m) for l in range(5) for m in range(-l, l + 1)]  # the 25 real Y_l^m, l <= 4


def fill_smooth(out: np.ndarray, xyz: np.ndarray, field_index: int, rows=None, harmonic=None) -> None:
    """Synthetic analytic field into ``out`` (rows ``rows`` or all), in row chunks.
    ``harmonic`` is the ``spherical_harmonic(l, m, xyz)`` to use (default: this package's;
    the reference arm passes the reference's own, analytic.py:35)."""
    if harmonic is None:
        from paper_1908_07038_b200.analytic import spherical_harmonic as harmonic

    from concurrent.futures import ThreadPoolExecutor

    L = out.shape[1]
    cols = [(field_index * L + k) % 25 for k in range(L)]
    fac = 1.0 + np.arange(L) / L
    idx = np.arange(len(xyz)) if rows is None else rows

    def chunk(s):  # numpy releases the GIL in these ufuncs and copies
        r = slice(s, min(s + 65536, len(idx))) if rows is None else idx[s:s + 65536]
        basis = np.stack([harmonic(l, m, xyz[r]) for l, m in HARMONICS], axis=1)
        if rows is None:
            np.multiply(basis[:, cols], fac, out=out[r])
        else:
            out[r] = basis[:, cols] * fac

    with ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(chunk, range(0, len(idx), 65536)))


def workload_config(source, target, L, F, method, m, n, nparts=1, partitioner="blocks"):
    """The ``config`` dict both arms print (identical for the same workload)."""
    kind = "structured-bilinear" if method == "bilinear" else "FE"
    nbytes = (n + m) * L * 8 * F
    return {"workload": f"{source}->{target} {kind} remap apply, {L} levels x {F} field(s), P={nparts}",
            "levels": L, "fields": F, "targets": m, "source_nodes": n,
            "parallelism": "single device" if nparts == 1 else f"domain decomposition x{nparts} ({partitioner})",
            "l2": (f"inputs {nbytes / 1e9:.1f} GB > 126 MB L2 (no flush needed)" if nbytes > 126e6 else
                   f"inputs {nbytes / 1e6:.1f} MB fit in the 126 MB L2 (L2-resident timing)")}


def setup_remap(sg, source, target, nparts, rank, ctx, method="fe", partitioner="blocks"):
    from paper_1908_07038_b200.partition import PARTITIONERS

    S, T = sg.grid_from_name(source), sg.grid_from_name(target)
    dist = PARTITIONERS[partitioner](S, nparts)
    mesh = sg.generate_mesh(S, dist, rank, halo=2, include_pole=True)  # cli.py:131
    fs = sg.NodeColumns(mesh, ctx)
    tdist = sg.matching_partition(T, S, dist)
    if method == "bilinear":
        w = sg.build_bilinear(fs, T, tdist, ctx)
    else:
        w = sg.build_remap(fs, T, tdist, ctx)
    return S, T, mesh, fs, tdist, w


def cpu_apply(nodes, weights, src, out, nthreads):
    """The reference's apply expression (interp.py:219-223) — the oracle port — over target
    chunks on ``nthreads`` threads (numpy releases the GIL in gathers and ufuncs)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    m = len(nodes)
    chunk = 16384

    def job(s):
        sl = slice(s, min(s + chunk, m))
        out[sl] = O.apply_remap_k(nodes[sl], weights[sl], src)

    if nthreads <= 1:
        for s in range(0, m, chunk):
            job(s)
        return
    with ThreadPoolExecutor(nthreads) as ex:
        list(ex.map(job, range(0, m, chunk)))


def algorithmic_bytes(U, m, L, F, k=3):
    """F·(U·L·8 + m·L·8) + m·k·(4 + 8), k = stencil points."""
    return F * (U * L * 8 + m * L * 8) + m * k * 12


# ------------------------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def loaded_repo_libraries():
    """Shared objects under this repo mapped into the process (evidence of what ran)."""
    try:
        with open("/proc/self/maps") as fh:
            paths = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT + os.sep))


def import_reference():
    """The unmodified reference package installed into baseline/_ref by
    tools/install_reference.sh (pip --target of /root/reference/pkg).  Nothing of this repo's
    package is imported on this path."""
    if not os.path.isdir(os.path.join(REF_DIR, "spheregrid")):
        return None, f"reference not installed: {REF_DIR}/spheregrid missing (run tools/install_reference.sh)"
    sys.path.insert(0, REF_DIR)
    import spheregrid as R

    if not os.path.abspath(R.__file__).startswith(REF_DIR):
        return None, f"spheregrid resolved to {R.__file__}, not baseline/_ref"
    return R, None


def reference_threaded(R, nodes, weights, src_hosts, n, L, expect, reps=2):
    """The reference's own ``apply_remap`` (interp.py:206-228) with every host thread: the
    targets split into one contiguous chunk per thread, each chunk a reference
    ``InterpolationWeights`` + target ``Field`` whose host array is a view into one output,
    all chunks run at once from a thread pool — as the reference's ``run_ranks`` threads would
    run their ranks' applies (numpy releases the GIL in its gathers and ufuncs).  Returns
    (best seconds per step, threads, bitwise equal to ``expect``)."""
    from concurrent.futures import ThreadPoolExecutor

    m = len(nodes)
    nt = max(1, min(os.cpu_count() or 1, 64))
    bounds = np.linspace(0, m, nt + 1).astype(np.int64)
    out = np.empty((m, L))
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        RW = R.InterpolationWeights(target_global=np.arange(a, b, dtype=np.int64),
                                    nodes=np.ascontiguousarray(nodes[a:b], np.int64),
                                    weights=np.ascontiguousarray(weights[a:b]), fallback=np.zeros(b - a, bool),
                                    source_nnodes=n)
        parts.append((RW, R.Field(name="dst", shape=(int(b - a), L), kind=R.Kind.REAL64, host=out[a:b])))
    srcs = [R.Field(name=f"src{f}", shape=(n, L), kind=R.Kind.REAL64, host=h) for f, h in enumerate(src_hosts)]

    def step(ex):
        for sf in srcs:
            list(ex.map(lambda pr: R.apply_remap(pr[0], sf, pr[1]), parts))

    times = []
    with ThreadPoolExecutor(nt) as ex:
        step(ex)  # warm-up
        for _ in range(reps):
            t = time.perf_counter()
            step(ex)
            times.append(time.perf_counter() - t)
    return min(times), nt, bool(np.array_equal(out.view(np.uint64), expect.view(np.uint64)))


def run_reference(args):
    """--impl reference: the reference's OWN code path on this host, rank 0 only.

    Grids, latitudes, mesh, function spaces and fields come from the unmodified reference
    (``grid_from_name`` gaussian.py:37-62 / grid.py:127-145, ``generate_mesh`` mesh.py:229-338,
    ``NodeColumns`` / ``StructuredColumns`` / ``create_field``), and the timed step is the
    reference's ``apply_remap(weights, source_field, target_field)`` (interp.py:206-228),
    as the reference runs it: numpy on one core.  Only the stencils do not come from the
    reference's ``build_remap`` (its per-target Python loop takes ~2 h at O1280->O640,
    SURVEY.md §8(d)): they come from the oracle's restatement of the same search
    (``oracle.locate_kdtree``: scipy cKDTree k=8/32 candidates scored with the reference's
    arithmetic, interp.py:90-117; batched dgesv weights, interp.py:61-71), wrapped in the
    reference's own ``InterpolationWeights``.  libsgb200 is never loaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    source, target, L, F, method = config(args.config)
    R, why = import_reference()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    from oracle import oracle as O

    t0 = time.time()
    S, T = R.grid_from_name(source), R.grid_from_name(target)
    dist = R.blocks_partition(S, 1)
    mesh = R.generate_mesh(S, dist, 0, halo=2, include_pole=True)  # cli.py:131
    fs = R.NodeColumns(mesh, None)
    tdist = R.blocks_partition(T, 1)  # == matching_partition at P=1 (every target in part 0)
    tfs = R.StructuredColumns(T, tdist, 0)
    log(f"reference grids + mesh {time.time() - t0:.1f}s ({mesh.nb_nodes} nodes)")
    conn = mesh.element_connectivity
    txyz = T.xyz()
    stencils = "oracle.locate_kdtree + batched dgesv (reference build_remap takes ~2 h here)"
    if method == "bilinear":
        nodes, weights, _ = O.bilinear_stencil(S.latitudes, S.nlons, T.lonlats(), True)
        stencils = "oracle.bilinear_stencil (no reference method)"
    elif T.npts <= 20000:  # small configs: the reference's own build_remap (~4 ms per target)
        rw = R.build_remap(fs, T, tdist)
        nodes, weights = rw.nodes, rw.weights
        stencils = "reference build_remap (interp.py:154-203)"
    else:
        elem, nodes = O.locate_kdtree(mesh.node_xyz, conn.offsets, conn.indices, txyz)
        if (elem < 0).any():
            raise SystemExit("reference arm: target not located")
        weights = O.barycentric_weights_batched(mesh.node_xyz, nodes, txyz)
    m = len(nodes)
    W = R.InterpolationWeights(target_global=tfs.local_points, nodes=np.ascontiguousarray(nodes, np.int64),
                               weights=np.ascontiguousarray(weights), fallback=np.zeros(m, bool),
                               source_nnodes=mesh.nb_nodes, source_global=mesh.node_global)
    from spheregrid.analytic import spherical_harmonic as ref_harmonic

    srcs, dsts = [], []
    for f in range(F):
        sf = fs.create_field(f"src{f}", levels=L)
        fill_smooth(sf.host, mesh.node_xyz, f, harmonic=ref_harmonic)
        srcs.append(sf)
        dsts.append(tfs.create_field(f"dst{f}", levels=L))
    log(f"reference setup {time.time() - t0:.1f}s")
    for _ in range(args.warmup):
        for sf, df in zip(srcs, dsts):
            R.apply_remap(W, sf, df)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        for sf, df in zip(srcs, dsts):
            R.apply_remap(W, sf, df)
        times.append(time.perf_counter() - t)
    units = m * L * F
    ms = 1e3 * sum(times) / len(times)
    value = units / (ms * 1e-3) / 1e9
    t_thr, nthr, thr_ok = reference_threaded(R, W.nodes, W.weights, [sf.host for sf in srcs], mesh.nb_nodes, L,
                                             dsts[-1].host)
    line = {
        "metric": metric_name(source, target, method, L), "value": value, "unit": "Gpts·lev/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic spherical harmonics)",
        "impl": "reference",
        "config": workload_config(source, target, L, F, method, m, mesh.nb_nodes, args.gpus, args.partitioner),
        "reference": {"package": os.path.relpath(os.path.dirname(R.__file__), ROOT), "version": R.__version__,
                      "timed": "spheregrid.apply_remap(InterpolationWeights, Field, Field) per field (interp.py:206-228)",
                      "built_by_reference": "grid_from_name, generate_mesh, NodeColumns, StructuredColumns, "
                                            "create_field, InterpolationWeights, analytic.spherical_harmonic",
                      "stencils": stencils,
                      "setup_s": round(time.time() - t0, 1),
                      "repo_libraries_loaded": loaded_repo_libraries(),
                      "product_imported": "paper_1908_07038_b200" in sys.modules},
        "cpu_baseline": {"value": value, "unit": "Gpts·lev/s", "cores": 1, "kind": "reference",
                         "sample": f"full {source}->{target} apply x{F} field(s) per step: the reference's own "
                                   "apply_remap (numpy, single-threaded as the reference runs it at P=1)"},
        "threaded": {"value": units / t_thr / 1e9, "unit": "Gpts·lev/s", "cores": nthr, "bitwise_vs_1_core": thr_ok,
                     "sample": f"the same step with {nthr} host threads: the reference's own apply_remap on "
                               f"{nthr} contiguous target chunks at once (as its run_ranks threads would run "
                               "P ranks; numpy releases the GIL), best of 2 — reported beside the 1-core value"},
        "e2e": {"value": value, "unit": "Gpts·lev/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def emulated_halo(sg, S, L, flush, parts=8, halo=2, partitioner="equal_regions", reps=5):
    """The halo exchange of the N>1 step at one point of cfg4 (BASELINE configs[3]), emulated
    on ONE GPU: every rank's field lives in this GPU's HBM and each rank's fused pull kernel
    (pack + transfer + unpack in one pass over peer pointers) is timed on its own, with L2
    flushed before every launch by an apply of the main workload.  On P GPUs the ranks run
    concurrently and the peer reads cross NVLink, so the exchange time there is the max over
    ranks of NVLink-bound pulls; here it is the max over ranks of HBM-bound pulls."""
    from paper_1908_07038_b200.device import DeviceArray, Event
    from paper_1908_07038_b200.partition import PARTITIONERS

    dist = PARTITIONERS[partitioner](S, parts)
    meshes = [sg.generate_mesh(S, dist, r, halo=halo, include_pole=True) for r in range(parts)]
    plans = sg.run_ranks(parts, lambda ctx: sg.NodeColumns(meshes[ctx.rank], ctx).exchange_plan, devices=[0])
    fields = [DeviceArray(m.nb_nodes, L, np.float64) for m in meshes]
    info = [(d.ptr, d.pitch, d.device) for d in fields]
    ms, nbytes = [], []
    for r in range(parts):
        plans[r].pull(fields[r], info)
        t = []
        for _ in range(reps):
            flush()
            e0, e1 = Event(0), Event(0)
            e0.record()
            plans[r].pull(fields[r], info)
            e1.record()
            t.append(Event.elapsed_ms(e0, e1))
        ms.append(statistics.median(t))
        nbytes.append(sum(len(v) for v in plans[r].recv.values()) * L * 8)
    # all ranks' signalled pulls (the N>1 exchange kernel, csrc/step.cu) as ONE launch
    from paper_1908_07038_b200.execute import emulated_exchanges, launch_exchanges

    xs = emulated_exchanges(list(zip(plans, fields)))
    launch_exchanges(xs)
    t = []
    for _ in range(reps):
        flush()
        e0, e1 = Event(0), Event(0)
        e0.record()
        launch_exchanges(xs)
        e1.record()
        t.append(Event.elapsed_ms(e0, e1))
    one = statistics.median(t)
    epochs = [x.check() for x in xs]
    del xs
    for d in fields:
        d.close()
    worst = max(ms)
    return {"bytes_per_exchange": int(sum(nbytes)), "worst_rank_pull_ms": worst,
            "signalled_one_launch_ms": one, "signalled_one_launch_GB_per_s": sum(nbytes) / (one * 1e-3) / 1e9,
            "signalled_epochs": epochs,
            "worst_rank_bytes": int(nbytes[int(np.argmax(ms))]), "per_rank_ms": [round(x, 4) for x in ms],
            "scope": f"cfg4 point O1280, {L} lev, halo {halo}, {partitioner} P={parts}, EMULATED on one GPU: "
                     "all ranks' fields in this GPU's HBM, each rank's pull kernel timed alone with L2 "
                     "flushed (worst_rank_pull_ms = max over ranks; not concurrent), and all ranks' signalled "
                     "pulls as ONE launch (signalled_one_launch_*, concurrent). HBM, not NVLink (needs >1 GPU)"}


def emulated_fused_step(sg, source, target, L, parts=8, partitioner="equal_regions", reps=10):
    """The N>1 fused step (csrc/step.cu: exchange over peer memory + apply, device-side ready /
    done signals, one kernel per rank) for ``parts`` ranks EMULATED on one GPU as ONE launch
    over every rank's data (ranks whose kernels wait on each other must not be separate
    launches on one GPU).  Compared with the same ranks' work as plain apply launches over
    pre-exchanged fields (interior + boundary targets, one launch per rank, summed): the
    difference is what the fused exchange and the signalling cost.  Parity: every rank's
    target rows bitwise against the oracle apply (interp.py:219-223) on the analytic field."""
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, Event
    from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps
    from paper_1908_07038_b200.interp import apply_remap_range
    from paper_1908_07038_b200.partition import PARTITIONERS

    S, T = sg.grid_from_name(source), sg.grid_from_name(target)
    dist = PARTITIONERS[partitioner](S, parts)
    td = sg.matching_partition(T, S, dist)

    def prog(ctx):
        mesh = sg.generate_mesh(S, dist, ctx.rank, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        return mesh, fs.exchange_plan, sg.build_remap(fs, T, td, ctx)

    built = sg.run_ranks(parts, prog, devices=[0])
    ranks, full = [], []
    for mesh, plan, w in built:
        host = np.zeros((mesh.nb_nodes, L))
        fill_smooth(host, mesh.node_xyz, 0, rows=np.arange(mesh.nb_owned_nodes))
        src = DeviceArray(mesh.nb_nodes, L, np.float64)
        src.upload(host)
        ranks.append((w, plan, src, DeviceArray(len(w), L, np.float64)))
    steps = emulated_fused_steps(ranks)
    for _ in range(3):
        launch_fused_steps(steps)
    e0, e1 = Event(0), Event(0)
    e0.record()
    for _ in range(reps):
        launch_fused_steps(steps)
    e1.record()
    fused_ms = Event.elapsed_ms(e0, e1) / reps
    epochs = [st.check() for st in steps]
    # parity of the fused result, then the plain applies over exchanged fields for comparison
    ok = True
    for (w, plan, src, dst), (mesh, _, _) in zip(ranks, built):
        exp_src = np.empty((mesh.nb_nodes, L))
        fill_smooth(exp_src, mesh.node_xyz, 0)
        exp = O.apply_remap_k(w.nodes, w.weights, exp_src)
        ok &= bool(np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64)))
    info = [(r[2].ptr, r[2].pitch, 0) for r in ranks]
    for (w, plan, src, dst) in ranks:
        plan.pull(src, info)
    for _ in range(3):
        for (w, plan, src, dst) in ranks:
            apply_remap_range(w, [src], [dst], 0, len(w), 0, 0)
    e0.record()
    for _ in range(reps):
        for (w, plan, src, dst) in ranks:
            apply_remap_range(w, [src], [dst], 0, len(w), 0, 0)
    e1.record()
    plain_ms = Event.elapsed_ms(e0, e1) / reps
    m_tot = sum(len(r[0]) for r in ranks)
    nbound = sum(st.n_boundary for st in steps)
    ghost_bytes = sum(sum(len(v) for v in r[1].recv.values()) for r in ranks) * L * 8
    for r in ranks:
        r[2].close()
        r[3].close()
    return {"parts": parts, "partitioner": partitioner, "halo": 2, "targets": m_tot, "boundary_targets": nbound,
            "ghost_bytes_per_exchange": ghost_bytes, "fused_step_ms": fused_ms,
            "plain_apply_ms": plain_ms, "overhead_ms": fused_ms - plain_ms,
            "Gpts_lev_per_s": m_tot * L / (fused_ms * 1e-3) / 1e9, "epochs": epochs,
            "target_rows_bitwise": ok,
            "scope": f"{source}->{target}, {L} lev: {parts} ranks EMULATED on one GPU as ONE launch of the fused "
                     "step (signal kernel + step kernel over all ranks' data, ghost rows read from the owners' "
                     "fields, ready/done words in HBM) vs the same ranks as one plain apply launch each over "
                     "fields whose ghosts were exchanged beforehand; not NVLink (needs >1 GPU)"}


def run_single(args):
    import paper_1908_07038_b200 as sg
    from paper_1908_07038_b200.device import DeviceArray, Event, PinnedArray

    source, target, L, F, method = config(args.config)
    dev = 0
    sg.set_device(dev)
    t0 = time.time()
    S, T, mesh, fs, tdist, w = setup_remap(sg, source, target, 1, 0, None, method)
    m, n = len(w), mesh.nb_nodes
    U = w.distinct_sources()
    log(f"setup {time.time() - t0:.1f}s: {n} source nodes, {m} targets, U={U}")
    # host inputs in pinned memory (also the e2e inputs)
    hsrc = [PinnedArray((n, L)) for _ in range(F)]
    hdst = [PinnedArray((m, L)) for _ in range(F)]
    for f in range(F):
        fill_smooth(hsrc[f].array, mesh.node_xyz, f)
    dsrc = [DeviceArray(n, L, np.float64) for _ in range(F)]
    ddst = [DeviceArray(m, L, np.float64) for _ in range(F)]
    for f in range(F):
        dsrc[f].upload(hsrc[f].array)
    log(f"inputs ready {time.time() - t0:.1f}s")

    clocks = ClockSampler(dev)
    clocks.start()
    # ---- device-resident timing: one apply launch per step, events around every launch ----
    for _ in range(args.warmup):
        sg.apply_remap_device(w, dsrc, ddst, variant=args.variant)
    sg.synchronize(dev)
    ev = [Event(dev) for _ in range(args.steps + 1)]
    clocks.active = True
    ev[0].record()
    for k in range(args.steps):
        sg.apply_remap_device(w, dsrc, ddst, variant=args.variant)
        ev[k + 1].record()
    sg.synchronize(dev)
    launch_ms = [Event.elapsed_ms(ev[k], ev[k + 1]) for k in range(args.steps)]
    total_ms = Event.elapsed_ms(ev[0], ev[-1])
    clocks.active = False
    ms = total_ms / args.steps
    ms_median = statistics.median(launch_ms)
    units = m * L * F
    value = units / (ms * 1e-3) / 1e9
    device_out = ddst[F - 1].to_numpy()  # checked against the CPU baseline's result below

    # ---- PCIe h2d peak on this box (the e2e path's roofline): one 2 GiB pinned DMA ----------
    prow = (2 << 30) // (L * 8)
    pdev = DeviceArray(prow, L, np.float64)
    phost = PinnedArray((prow, L))
    phost.array[:] = 1.0
    pcie = []
    for _ in range(3):
        p0, p1 = Event(dev), Event(dev)
        p0.record()
        pdev.upload(phost.array, sync=False)
        p1.record()
        pcie.append(prow * L * 8 / (Event.elapsed_ms(p0, p1) * 1e-3) / 1e9)
    pcie_h2d_gbs = max(pcie)
    del pdev, phost

    # ---- e2e through the public API: host fields in pinned memory -------------------------
    import paper_1908_07038_b200.interp as sgi

    sgi.HOST_EXECUTE_MODE = args.e2e_mode
    sgi.HOST_EXECUTE_CHUNKS = args.e2e_chunks
    if args.e2e_period >= 0:
        sgi.HOST_EXECUTE_DIRECT_PERIOD = args.e2e_period
    fsrc = [sg.Field(name=f"src{f}", shape=(n, L), kind=sg.Kind.REAL64, host=hsrc[f].array) for f in range(F)]
    fdst = [sg.Field(name=f"dst{f}", shape=(m, L), kind=sg.Kind.REAL64, host=hdst[f].array) for f in range(F)]
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(4):  # warm: staging buffers, pipeline plans (auto: gather for pinned sources)
        sg.apply_remap_fields(w, fsrc, fdst)
    clocks.active = True
    e2e_times = []
    for _ in range(e2e_steps):
        t = time.perf_counter()
        sg.apply_remap_fields(w, fsrc, fdst)  # all F fields in one pipelined call
        e2e_times.append(time.perf_counter() - t)
    e2e_s = statistics.median(e2e_times)
    clocks.active = False
    clocks.stop()

    halo = fstep = None
    if args.config == "cfg3" and not args.no_halo:
        try:  # auxiliary evidence: never lose the bench line over it
            halo = emulated_halo(sg, S, L, lambda: sg.apply_remap_device(w, dsrc, ddst, variant=args.variant))
        except Exception as exc:  # noqa: BLE001
            halo = {"error": f"{type(exc).__name__}: {exc}"}
        try:
            fstep = emulated_fused_step(sg, source, target, L)
        except Exception as exc:  # noqa: BLE001
            fstep = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- CPU baseline, 1 core, same workload: the reference's own apply_remap (baseline/_ref)
    # on the same stencils and host arrays when installed, else the oracle port of
    # interp.py:219-223; its result (last field) is also the parity check of the device and
    # e2e outputs ------------------------------------------------------------------------
    cpu = None
    parity = {"checked": False}
    if not args.no_cpu_baseline:
        out = np.empty((m, L))
        R, _ = import_reference()
        if R is not None:
            RW = R.InterpolationWeights(target_global=np.arange(m, dtype=np.int64), nodes=w.nodes.astype(np.int64),
                                        weights=w.weights, fallback=np.zeros(m, bool), source_nnodes=n)
            rsrc = [R.Field(name=f"src{f}", shape=(n, L), kind=R.Kind.REAL64, host=hsrc[f].array) for f in range(F)]
            rdst = R.Field(name="dst", shape=(m, L), kind=R.Kind.REAL64, host=out)

            def cpu_step():
                for f in range(F):
                    R.apply_remap(RW, rsrc[f], rdst)
            kind, what = "reference", "the reference's own apply_remap (baseline/_ref, interp.py:206-228)"
        else:
            def cpu_step():
                for f in range(F):
                    cpu_apply(w.nodes, w.weights, hsrc[f].array, out, 1)
            kind, what = "port", "the oracle port of interp.py:219-223 (baseline/_ref not installed)"
        times = []
        for _ in range(2):
            tt = time.perf_counter()
            cpu_step()
            times.append(time.perf_counter() - tt)
        cpu = {"value": units / min(times) / 1e9, "unit": "Gpts·lev/s", "cores": 1, "kind": kind,
               "sample": f"full {source}->{target} apply x{F} field(s), best of 2: {what}, numpy single-threaded "
                         "as the reference runs it"}
        if R is not None:
            t_thr, nthr, thr_ok = reference_threaded(R, w.nodes, w.weights, [h.array for h in hsrc], n, L, out)
            cpu["threaded"] = {"value": units / t_thr / 1e9, "unit": "Gpts·lev/s", "cores": nthr,
                               "bitwise_vs_1_core": thr_ok,
                               "sample": f"the reference's own apply_remap on {nthr} target chunks from {nthr} "
                                         "threads at once (numpy releases the GIL), best of 2"}
        parity = {"checked": True, "against": kind,
                  "device_bitwise_vs_cpu": bool(np.array_equal(device_out.view(np.uint64), out.view(np.uint64))),
                  "e2e_bitwise_vs_cpu": bool(np.array_equal(hdst[F - 1].array.view(np.uint64), out.view(np.uint64)))}
        if method == "fe":  # the stencils of the timed kernel vs the reference's search and solver
            from oracle import oracle as O

            t0s = time.perf_counter()
            conn = mesh.element_connectivity
            txyz = T.xyz()[w.target_global]
            e_o, c_o = O.locate_kdtree(mesh.node_xyz, conn.offsets, conn.indices, txyz)
            ow = O.barycentric_weights_batched(mesh.node_xyz, c_o, txyz)
            parity.update({
                "stencils_bitwise_vs_reference_search": bool((e_o >= 0).all() and np.array_equal(w.nodes, c_o)),
                "weights_bitwise_vs_reference_dgesv": bool(np.array_equal(w.weights.view(np.uint64),
                                                                          ow.view(np.uint64))),
                "stencil_check": "every target: oracle.locate_kdtree (the reference's cKDTree k=8/32 candidates "
                                 "and scoring) + np.linalg.solve, as interp.py:102-117 / 61-71",
                "stencil_check_s": round(time.perf_counter() - t0s, 1)})

    h2d_moved = int(w.__dict__.get("last_host_rows_moved", n)) * L * 8 * F
    peak, peak_src = measured_peak()
    B = algorithmic_bytes(U, m, L, F, w.nodes.shape[1])
    kern_ms = statistics.mean(launch_ms)
    achieved = B / (kern_ms * 1e-3) / 1e9
    line = {
        "metric": metric_name(source, target, method, L), "value": value, "unit": "Gpts·lev/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": ms_median, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic spherical harmonics)",
        "config": workload_config(source, target, L, F, method, m, n),
        "kernel": {"variant": args.variant, "distinct_sources": U},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.config), "algorithmic_bytes_per_launch": B,
                     "kernel_ms": kern_ms, "peak_source": peak_src},
        "e2e": {"value": units / e2e_s / 1e9, "unit": "Gpts·lev/s",
                "h2d_bytes_per_step": h2d_moved,
                "input_bytes_per_step": n * L * 8 * F,
                "d2h_bytes_per_step": m * L * 8 * F, "ms_per_step": e2e_s * 1e3, "statistic": "median",
                "ms_per_step_mean": 1e3 * sum(e2e_times) / len(e2e_times),
                "api": "paper_1908_07038_b200.apply_remap_fields(weights, host Fields, host Fields)",
                "roofline": {"bound": "pcie h2d", "achieved": h2d_moved / e2e_s / 1e9, "peak": pcie_h2d_gbs,
                             "unit": "GB/s", "frac": h2d_moved / e2e_s / 1e9 / pcie_h2d_gbs,
                             "peak_source": "measured here: 2 GiB pinned h2d DMA, best of 3",
                             "note": "source rows that must cross PCIe each step / step time; the d2h of the "
                                     "target rows runs concurrently in the other direction"},
                "mode": args.e2e_mode, "chunks": args.e2e_chunks, "direct_period": args.e2e_period,
                "auto_trials_s": {k: [round(x, 4) for x in v] for k, v in w.__dict__.get("_auto_s", {}).items()}},
        "halo_emulated": halo,
        "fused_step_emulated": fstep,
        "cpu_baseline": cpu,
        "gpu_launches": args.steps,
        "parity": parity,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    log(f"total {time.time() - t0:.1f}s")


# ------------------------------------------------------------------------------------------
def run_multi(args):
    """N > 1: one process per GPU (torchrun).  Step = source-field halo exchange (pack ->
    grouped NCCL send/recv -> unpack, on its own stream) overlapped with the apply of the
    interior targets, then the boundary targets; the step is one captured CUDA graph."""
    import torch
    import torch.distributed as dist

    import paper_1908_07038_b200 as sg
    from paper_1908_07038_b200.device import Event, PinnedArray
    from paper_1908_07038_b200.execute import DistributedRemap

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ndev = sg._native.device_count()
    dev = local % max(ndev, 1)
    sg.set_device(dev)
    local = dev
    ctx = sg.DistContext(device=local, transport=args.transport)
    # one GPU per rank? (device UUIDs, not the visible-device count: a launcher may give each
    # process only its own GPU)
    own_gpu = len(set(ctx.share(sg._native.device_uuid(local)))) == world
    if not own_gpu and args.transport == "nccl":
        raise SystemExit(f"{world} ranks share GPUs: NCCL needs one GPU per rank (use --transport ipc)")
    source, target, L, F, method = config(args.config)
    t0 = time.time()
    S, T, mesh, fs, tdist, w = setup_remap(sg, source, target, world, rank, ctx, method, args.partitioner)
    m, n = len(w), mesh.nb_nodes
    n_owned = mesh.nb_owned_nodes
    hsrc = PinnedArray((n, L))
    hsrc.array[:] = 0.0
    fill_smooth(hsrc.array, mesh.node_xyz, 0, rows=np.arange(n_owned))
    hdst = PinnedArray((m, L))
    f = sg.Field(name="src", shape=(n, L), kind=sg.Kind.REAL64, host=hsrc.array).allocate_device()
    tf = sg.Field(name="dst", shape=(m, L), kind=sg.Kind.REAL64, host=hdst.array).allocate_device()
    def allreduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return t.tolist()

    fallback, err = None, ""
    try:  # a failed peer mapping raises on every rank together (DistContext._all_or_none)
        run = DistributedRemap(fs, w, ctx, f.device, tf.device, variant=args.variant, fused=args.fused)
    except sg.SpheregridError as exc:
        if not own_gpu:
            raise SystemExit(f"rank {rank}: peer memory unavailable and ranks share GPUs: {exc}")
        fallback = f"peer memory unavailable ({exc}); NCCL exchange + apply used"
        log(f"rank {rank}: {fallback}")
        args.transport = ctx.transport = "nccl"
        run = DistributedRemap(fs, w, ctx, f.device, tf.device, variant=args.variant, fused=False)
    try:
        run.step()
        run.synchronize()  # raises if a device-side wait of the fused step timed out
        ok = 1.0
    except sg.SpheregridError as exc:
        ok, err = 0.0, str(exc)
    if allreduce([ok], dist.ReduceOp.MIN)[0] == 0.0:
        if not args.fused:
            raise SystemExit(f"rank {rank}: first step failed: {err}")
        # explicit, reported: the line carries transport_fallback and step.fused = false
        fallback = f"fused step failed ({err or 'on another rank'}); exchange ({args.transport}) + apply used"
        log(f"rank {rank}: {fallback}")
        run = DistributedRemap(fs, w, ctx, f.device, tf.device, variant=args.variant, fused=False)
        run.step()
        run.synchronize()
    log(f"rank {rank}: setup {time.time() - t0:.1f}s, {n} nodes ({n_owned} owned), {m} targets, "
        f"interior targets {run.n_interior}, {sum(len(v) for v in fs.exchange_plan.recv.values())} ghosts")
    for _ in range(args.warmup):
        run.step()
    run.synchronize()
    try:
        if not run.stream_ordered:
            raise RuntimeError("host-synchronised transport")
        run.capture()
        for _ in range(2):
            run.step()
        run.synchronize()
        graphed = True
    except Exception as exc:  # noqa: BLE001 - eager fallback keeps the same kernels
        log(f"rank {rank}: graph capture failed ({exc}); eager steps")
        run.graph = None
        graphed = False
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        clocks.active = True
    ctx.barrier()
    e0, e1 = Event(local), Event(local)
    e0.record(run.main.stream)
    for _ in range(args.steps):
        run.step()
    e1.record(run.main.stream)
    run.synchronize()
    my_ms = Event.elapsed_ms(e0, e1)
    ctx.barrier()

    tmax = allreduce([my_ms], dist.ReduceOp.MAX)[0]
    msum = allreduce([float(m)], dist.ReduceOp.SUM)[0]
    # the dominant kernel alone: this rank's apply over all its targets (roofline per GPU)
    from paper_1908_07038_b200.interp import apply_remap_range

    ctx.barrier()
    k0, k1 = Event(local), Event(local)
    k0.record(run.main.stream)
    for _ in range(args.steps):
        apply_remap_range(w, [f.device], [tf.device], 0, m, args.variant, run.main.stream)
    k1.record(run.main.stream)
    run.synchronize()
    kern_ms = Event.elapsed_ms(k0, k1) / args.steps
    my_bytes = float(algorithmic_bytes(w.distinct_sources(), m, L, F, w.nodes.shape[1]))
    worst_kern_ms = allreduce([kern_ms], dist.ReduceOp.MAX)[0]
    worst_bytes = allreduce([my_bytes if kern_ms == worst_kern_ms else 0.0], dist.ReduceOp.MAX)[0]
    # halo exchange alone (bytes over NVLink)
    from paper_1908_07038_b200.parallel import _signalled_exchange

    def exchanger(plan, d, stream, transport=args.transport):
        """(run, device-timed?, label) of the halo exchange of ``plan`` on ``d`` (collective)."""
        if transport == "nccl":
            return (lambda: plan.exchange_nccl(d, ctx.nccl_comm(), stream)), True, "nccl pack/send/recv/unpack"
        if transport == "nvlink":
            try:
                x = _signalled_exchange(ctx, plan, d)
            except sg.SpheregridError:  # raised on every rank together: peer memory unavailable
                x = None
                if own_gpu:
                    return exchanger(plan, d, stream, "nccl")
            if x is not None:
                return (lambda: x.launch(stream)), True, "signalled pull over NVLink, one kernel per rank"
        return (lambda: ctx.device_exchange(plan, d, stream)), False, "pull kernel between host barriers"

    def time_exchange(run_x, timed, stream, reps):
        if timed:
            a0, a1 = Event(local), Event(local)
            a0.record(stream)
            for _ in range(reps):
                run_x()
            a1.record(stream)
            sg.synchronize(local, stream)
            return Event.elapsed_ms(a0, a1) / reps
        tt = time.perf_counter()
        for _ in range(reps):
            run_x()
        return (time.perf_counter() - tt) * 1e3 / reps

    ctx.barrier()
    hx, htimed, hlabel = exchanger(fs.exchange_plan, f.device, run.halo.stream)
    hx()
    sg.synchronize(local, run.halo.stream)
    ctx.barrier()
    halo_ms = time_exchange(hx, htimed, run.halo.stream, args.steps)
    send_bytes = float(sum(len(v) for v in fs.exchange_plan.send.values()) * L * 8)
    hmax = allreduce([halo_ms], dist.ReduceOp.MAX)[0]
    hsum = allreduce([send_bytes], dist.ReduceOp.SUM)[0]
    # e2e: the owned source rows this step needs (read by the rank's own stencils or sent to a
    # peer) host -> device, exchange + apply, target rows device -> host.  The pinned source is
    # mapped, so one kernel pulls the row runs over PCIe (sg_field_h2d_row_runs).
    from paper_1908_07038_b200.functionspace import row_runs

    nd = w.nodes[w.nodes < n_owned].ravel()
    sends = [np.asarray(v, np.int64) for v in fs.exchange_plan.send.values()]
    runs = row_runs(np.concatenate([nd] + sends))
    h2d_rows = int(runs[:, 1].sum()) if len(runs) else 0
    ctx.barrier()
    e2e_steps = max(3, min(args.steps, 10))
    tt = time.perf_counter()
    for _ in range(e2e_steps):
        f.device.upload_row_runs(hsrc.array, runs, stream=run.main.stream, sync=False)
        run.step()
        tf.device.download(hdst.array, stream=run.main.stream, sync=False)
        run.synchronize()
    my_e2e = (time.perf_counter() - tt) / e2e_steps
    ctx.barrier()
    e2e_max = allreduce([my_e2e], dist.ReduceOp.MAX)[0]
    h2d = allreduce([float(h2d_rows * L * 8)], dist.ReduceOp.SUM)[0]
    d2h = allreduce([float(m * L * 8)], dist.ReduceOp.SUM)[0]
    if clocks:
        clocks.active = False
        clocks.stop()

    # ---- parity: this rank's exchanged source rows and its target rows, bitwise, against a
    # single-process recomputation: the synthetic field evaluated on EVERY local row (the
    # ghosts' owners evaluate the same function at the same coordinates), then the oracle's
    # apply (interp.py:219-223) on this rank's stencils ------------------------------------
    from oracle import oracle as O

    exp_src = np.empty((n, L))
    fill_smooth(exp_src, mesh.node_xyz, 0)
    src_ok = bool(np.array_equal(f.device.to_numpy().view(np.uint64), exp_src.view(np.uint64)))
    dst_ok = bool(np.array_equal(tf.device.to_numpy().view(np.uint64),
                                 O.apply_remap_k(w.nodes, w.weights, exp_src).view(np.uint64)))
    e2e_ok = bool(np.array_equal(hdst.array.view(np.uint64), tf.device.to_numpy().view(np.uint64)))
    oks = allreduce([float(src_ok), float(dst_ok), float(e2e_ok)], dist.ReduceOp.MIN)
    parity = {"checked": True, "source_rows_bitwise": oks[0] == 1.0, "target_rows_bitwise": oks[1] == 1.0,
              "e2e_target_rows_bitwise": oks[2] == 1.0, "targets_checked": int(msum),
              "against": "per rank: analytic field on every local row (owned + ghost) and the oracle apply "
                         "(interp.py:219-223) on the rank's own stencils"}
    comm = {"transport": args.transport, "transport_fallback": fallback, "exchange": hlabel}
    if own_gpu:
        info = ctx.comm_info()
        nr = allreduce([float(info["nranks"])], dist.ReduceOp.MIN)[0]
        comm.update({"nccl_nranks": int(nr), "nccl_version": info["nccl_version"],
                     "rank0_cu_device": info["device"]})

    # ---- cfg4 (BASELINE configs[3]): NodeColumns halo exchange of the O1280 source at halo
    # widths 1..3, every rank at once, device timing, max over ranks --------------------------
    sweep = []
    if not args.no_halo_sweep:
        from paper_1908_07038_b200.device import DeviceArray, Stream
        from paper_1908_07038_b200.partition import PARTITIONERS

        dist_s = PARTITIONERS[args.partitioner](S, world)
        hs = Stream(local)
        for h in (1, 2, 3):
            mh = mesh if h == 2 else sg.generate_mesh(S, dist_s, rank, halo=h, include_pole=True)
            plan = sg.NodeColumns(mh, ctx).exchange_plan
            d = DeviceArray(mh.nb_nodes, L, np.float64, local)
            vals = mh.node_global[:, None].astype(np.float64) + np.arange(L)[None, :] / L
            init = np.where(mh.node_ghost[:, None], -1.0, vals)
            d.upload(init)

            rb = float(sum(len(v) for v in plan.recv.values()) * L * 8)
            tot = allreduce([rb], dist.ReduceOp.SUM)[0]
            entry = {"halo": h, "bytes_per_exchange": tot}
            # the transport of the run, then NCCL (the library baseline) when each rank has a GPU
            transports = [args.transport] + (["nccl"] if args.transport != "nccl" and own_gpu else [])
            for k, tr in enumerate(transports):
                d.upload(init)
                xrun, xtimed, xlabel = exchanger(plan, d, hs.stream, tr)
                xrun()
                sg.synchronize(local, hs.stream)
                ok = bool(np.array_equal(d.to_numpy(), vals))
                for _ in range(3):
                    xrun()
                sg.synchronize(local, hs.stream)
                ctx.barrier()
                ms_h = time_exchange(xrun, xtimed, hs.stream, args.steps)
                r = allreduce([ms_h, rb, float(len(plan.peers))], dist.ReduceOp.MAX)
                okmin = allreduce([float(ok)], dist.ReduceOp.MIN)[0]
                res = {"ms": r[0], "GB_per_s": tot / (r[0] * 1e-3) / 1e9, "worst_rank_recv_bytes": r[1],
                       "max_peers": int(r[2]), "ghosts_bitwise": okmin == 1.0, "exchange": xlabel,
                       "timing": "device events on the exchange stream, max over ranks" if xtimed
                       else "wall clock incl. host barriers, max over ranks"}
                if k == 0:
                    entry.update(res)
                else:
                    entry["nccl_baseline"] = res
            sweep.append(entry)
            d.close()

    if rank == 0:
        ms = tmax / args.steps
        units = msum * L
        value = units / (ms * 1e-3) / 1e9
        cfg = workload_config(source, target, L, 1, method, int(msum), int(S.npts + 2), world, args.partitioner)
        line = {
            "metric": metric_name(source, target, method, L), "value": value, "unit": "Gpts·lev/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic spherical harmonics)",
            "config": cfg,
            "step": {"description": (
                "fused exchange+apply: one signal kernel + one step kernel per rank; boundary targets read ghost "
                "rows from the owners' HBM (CUDA IPC over NVLink), ready/done flag words in peer memory, no "
                "host or NCCL barrier" if run.signalled else
                "fused exchange+apply over peer memory, host barriers (ranks share a GPU)" if run.fused else
                f"halo exchange ({args.transport}) + apply, interior targets overlapped when stream-ordered"),
                     "halo": 2, "cuda_graph": graphed, "transport": args.transport, "fused": bool(run.fused),
                     "device_signalled": bool(run.signalled)},
            "transport_fallback": fallback,
            "comm": comm,
            "parity": parity,
            "halo": {"bytes_per_exchange": hsum, "ms": hmax, "GB_per_s": hsum / (hmax * 1e-3) / 1e9},
            "halo_sweep": sweep,
            "roofline": {"bound": "hbm", "achieved": worst_bytes / (worst_kern_ms * 1e-3) / 1e9, "peak": measured_peak()[0],
                         "unit": "GB/s", "frac": worst_bytes / (worst_kern_ms * 1e-3) / 1e9 / measured_peak()[0],
                         "traffic": None, "kernel_ms": worst_kern_ms, "algorithmic_bytes_per_launch": worst_bytes,
                         "peak_source": measured_peak()[1],
                         "note": "apply kernel of the slowest rank over all its targets, timed alone"},
            "e2e": {"value": units / e2e_max / 1e9, "unit": "Gpts·lev/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_max * 1e3},
            "gpu_launches": run.launches_per_step * args.steps,
            "clocks": clocks.summary() if clocks else None,
        }
        print(json.dumps(line), flush=True)
    ctx.barrier()
    ctx.close_ipc()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--variant", type=int, default=0, help="apply kernel: 0 default, 1 warp LDG, 2 TMA bulk")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-halo", action="store_true", help="N=1: skip the one-GPU emulation of the cfg4 halo exchange")
    ap.add_argument("--e2e-chunks", type=int, default=0, help="host-execute pipeline depth (0 = auto)")
    ap.add_argument("--e2e-period", type=int, default=-1,
                    help="compact e2e: copy every n-th chunk directly instead of packing (-1 = library default)")
    ap.add_argument("--e2e-mode", default="auto", choices=["auto", "dma", "compact", "gather", "gather_warp", "zerocopy"],
                    help="host-buffer execute path for e2e (auto = GPU gather for page-locked sources, "
                         "else the faster of compact / dma timed on the first calls)")
    ap.add_argument("--partitioner", default="equal_regions", choices=["blocks", "equal_regions"],
                    help="N>1 source decomposition: equal regions (BASELINE configs[2]; EQ zonal "
                         "equal-area parts sized like blocks) or the reference pipeline's blocks bands")
    ap.add_argument("--fused", action=argparse.BooleanOptionalAction, default=True,
                    help="N>1 (default): no ghost copy — boundary targets read ghost rows from the owners' HBM "
                         "(CUDA IPC / NVLink) inside one step kernel per rank, fenced by device-side flag words "
                         "(one GPU per rank) or host barriers (ranks sharing a GPU); --no-fused: pack -> "
                         "transport -> unpack with the interior apply overlapped")
    ap.add_argument("--no-halo-sweep", action="store_true",
                    help="N>1: skip the cfg4 sweep (halo widths 1..3 exchanged on every rank)")
    ap.add_argument("--transport", default="nvlink", choices=["nvlink", "nccl", "ipc"],
                    help="N>1 halo exchange (cfg4 sweep, --no-fused steps): nvlink = one signalled pull "
                         "kernel per rank over CUDA-IPC mappings (ranks sharing a GPU: pull between host "
                         "barriers); nccl = pack -> NCCL send/recv -> unpack; ipc = pull between host barriers. "
                         "With nvlink the sweep also times NCCL as the library baseline")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    main()
