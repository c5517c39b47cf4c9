"""Generates the golden fixtures under tests/golden/ by running the UNMODIFIED reference
(`spheregrid`, /root/reference/pkg/src) in this container.  The reference cannot travel to
the GPU box, so its outputs are committed here as small .npz files.

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [names...]
Host check: tools/host_probe.py digests of numpy's arcsin/cos/sin/dot were identical here
and on the GPU box host (gpurun_out/probe_*.json), so coordinates built from these
latitudes have the same bits on both.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import spheregrid as R  # noqa: E402
from spheregrid import interp as RI  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


def latitudes():
    out = {}
    for n in [1, 2, 4, 8, 16, 32, 64, 80, 160, 320, 640, 1280]:
        t = time.time()
        out[f"n{n}"] = R.gaussian_latitudes(n)
        print("lat", n, round(time.time() - t, 1), flush=True)
    save("latitudes", **out)


def stencil_arrays(w):
    return dict(target_global=w.target_global, nodes=w.nodes.astype(np.int32), weights=w.weights,
                scale=w.scale, fallback=w.fallback)


def serial_remap(src, tgt, levels, fname):
    """P=1 pipeline slice (cli.py:129-144): mesh with poles, NodeColumns, build, apply on a
    random field (seed 2026, test_acceptance.py:133)."""
    S, T = R.grid_from_name(src), R.grid_from_name(tgt)
    dist = R.blocks_partition(S, 1)
    mesh = R.generate_mesh(S, dist, 0, halo=2, include_pole=True)
    fs = R.NodeColumns(mesh, None)
    tdist = R.matching_partition(T, S, dist)
    t = time.time()
    w = R.build_remap(fs, T, tdist)
    print(f"{fname} build_remap {time.time() - t:.1f} s", flush=True)
    f = fs.create_field("src", levels=levels)
    f.host[:] = np.random.default_rng(2026).normal(size=f.host.shape)
    tf = R.StructuredColumns(T, tdist, 0).create_field("dst", levels=levels)
    R.apply_remap(w, f, tf)
    save(fname, **stencil_arrays(w), src_lat=S.latitudes, tgt_lat=T.latitudes, node_global=mesh.node_global,
         out=tf.host)


def partitioned(src, tgt, nparts, halo, fname, levels=3):
    """Per-rank meshes, plans, halo payload bytes and stencils of the distributed pipeline."""
    S, T = R.grid_from_name(src), R.grid_from_name(tgt)
    captured = {}
    orig_send = R.RankContext.send

    def spy(self, dest, tag, payload):
        if tag == 102:
            captured[(self.rank, dest)] = bytes(payload)
        return orig_send(self, dest, tag, payload)

    def program(ctx):
        dist = R.blocks_partition(S, ctx.nranks)
        mesh = R.generate_mesh(S, dist, ctx.rank, halo=halo, include_pole=True)
        fs = R.NodeColumns(mesh, ctx)
        tdist = R.matching_partition(T, S, dist)
        f = fs.create_field("gid", levels=levels)
        owned = fs.owned_row_index()
        rng = np.random.default_rng(100 + ctx.rank)
        f.host[owned] = mesh.node_global[owned, None] * 1000.0 + np.arange(levels)[None, :] \
            + rng.normal(size=(len(owned), levels)) * 1e-3
        before = f.host.copy()
        sent0 = ctx.messages_sent
        fs.halo_exchange(f, ctx)
        msgs = ctx.messages_sent - sent0
        try:
            w = R.build_remap(fs, T, tdist, ctx)
            st = stencil_arrays(w)
            bad = -1
        except R.errors.NotLocated as e:
            st, bad = {}, e.target_global_index
        plan = fs.exchange_plan
        d = dict(node_global=mesh.node_global, node_part=mesh.node_part, node_remote=mesh.node_remote,
                 node_halo=mesh.node_halo, conn_off=mesh.element_connectivity.offsets,
                 conn_idx=mesh.element_connectivity.indices, elem_serial=mesh.elem_serial_id,
                 before=before, after=f.host, messages=np.int64(msgs), not_located=np.int64(bad),
                 tdist=tdist.part_of.astype(np.int8))
        for p, v in plan.send.items():
            d[f"send_{p}"] = v
        for p, v in plan.recv.items():
            d[f"recv_{p}"] = v
        for k, v in st.items():
            d["w_" + k] = v
        return d

    R.RankContext.send = spy
    try:
        t = time.time()
        res = R.run_ranks(nparts, program)
        print(f"{fname} {time.time() - t:.1f} s", flush=True)
    finally:
        R.RankContext.send = orig_send
    out = {"src_lat": S.latitudes, "tgt_lat": T.latitudes, "nparts": np.int64(nparts), "halo": np.int64(halo)}
    for r, d in enumerate(res):
        for k, v in d.items():
            out[f"r{r}_{k}"] = np.asarray(v)
    for (a, b), payload in captured.items():
        out[f"payload_{a}_{b}"] = np.frombuffer(payload, dtype=np.uint8)
    save(fname, **out)


def fallback_case():
    """halo 0: NotLocated with allow_fallback=False; fallback rows with True (interp.py:179-190)."""
    S, T = R.grid_from_name("O32"), R.grid_from_name("O16")
    out = {}

    def program(ctx):
        dist = R.blocks_partition(S, ctx.nranks)
        mesh = R.generate_mesh(S, dist, ctx.rank, halo=0, include_pole=True)
        fs = R.NodeColumns(mesh, ctx)
        tdist = R.matching_partition(T, S, dist)
        w = R.build_remap(fs, T, tdist, ctx, allow_fallback=True)
        try:
            R.build_remap(fs, T, tdist, ctx, allow_fallback=False)
            bad = -1
        except R.errors.NotLocated as e:
            bad = e.target_global_index
        return dict(bad=np.int64(bad), **stencil_arrays(w))

    res = R.run_ranks(4, program)
    for r, d in enumerate(res):
        for k, v in d.items():
            out[f"r{r}_{k}"] = np.asarray(v)
    save("fallback_O32_O16_p4_h0", **out)


def matching():
    out = {}
    for tgt, src, P in [("O16", "O32", 4), ("O80", "O160", 8), ("O160", "O320", 8), ("O640", "O1280", 8)]:
        S, T = R.grid_from_name(src), R.grid_from_name(tgt)
        t = time.time()
        idx, _ = R.PointCloudIndex(S).query(T.xyz())
        out[f"{tgt}_{src}_idx"] = idx.astype(np.int32)
        out[f"{tgt}_{src}_p{P}"] = R.matching_partition(T, S, R.blocks_partition(S, P)).part_of.astype(np.int8)
        print("matching", tgt, src, round(time.time() - t, 1), flush=True)
    save("matching", **out)


def o1280_sample(n_random=5000):
    """O1280 -> O640 serial: reference MeshLocator.locate on every lon 0/90/180/270 target
    plus random targets (SURVEY.md §7 'Golden generation at O1280')."""
    S, T = R.grid_from_name("O1280"), R.grid_from_name("O640")
    t = time.time()
    mesh = R.generate_mesh(S, R.blocks_partition(S, 1), 0, halo=2, include_pole=True)
    print("mesh", round(time.time() - t, 1), flush=True)
    loc = RI.MeshLocator(mesh)
    print("locator", round(time.time() - t, 1), flush=True)
    ll = T.lonlats()
    special = np.flatnonzero(np.isin(ll[:, 0], [0.0, 90.0, 180.0, 270.0]))
    rng = np.random.default_rng(1280)
    rand = rng.choice(T.npts, size=n_random, replace=False)
    ids = np.unique(np.concatenate([special, rand])).astype(np.int64)
    xyz = T.xyz()
    corners = np.empty((len(ids), 3), np.int64)
    weights = np.empty((len(ids), 3))
    for k, g in enumerate(ids):
        _, tri, c = loc.locate(xyz[g])
        corners[k] = c
        weights[k] = RI.barycentric_weights(tri, xyz[g])
    print("located", len(ids), round(time.time() - t, 1), flush=True)
    save("o1280_o640_sample", ids=ids, corners=corners.astype(np.int32), weights=weights,
         src_lat=S.latitudes, tgt_lat=T.latitudes)


def checksums():
    """checksum (functionspace.py:233-254) of fields scattered over P ranks: the digest is
    partition-invariant; also the NodeColumns (mesh halo 1) variant."""
    out = {}
    for name, kind, levels in [("O32", R.Kind.REAL64, 3), ("F8", R.Kind.INT64, 2), ("O16", R.Kind.REAL32, 5)]:
        g = R.grid_from_name(name)
        rng = np.random.default_rng(77)
        vals = rng.normal(size=(g.npts, levels))
        if kind is R.Kind.INT64:
            vals = rng.integers(-10**12, 10**12, size=(g.npts, levels))
        vals = vals.astype(kind.dtype)
        for P in (1, 2, 4):
            def program(ctx):
                dist = R.blocks_partition(g, ctx.nranks)
                fs = R.StructuredColumns(g, dist, ctx.rank)
                f = fs.create_field("x", levels, kind)
                c = ctx if ctx.nranks > 1 else None
                R.scatter_field(fs, f, c, vals if ctx.rank == 0 else None)
                d1 = R.checksum(fs, f, c)
                mesh = R.generate_mesh(g, dist, ctx.rank, halo=1, include_pole=False)
                nfs = R.NodeColumns(mesh, c)
                nf = nfs.create_field("y", levels, kind)
                own = nfs.owned_row_index()
                nf.host[own] = vals[mesh.node_global[own]]
                d2 = R.checksum(nfs, nf, c)
                return d1, d2
            res = R.run_ranks(P, program)
            out[f"{name}_p{P}"] = np.array([res[0][0], res[0][1]], dtype=np.uint64)
        out[f"{name}_values"] = vals
    save("checksum", **out)


def rotated():
    """Rotated lon-lat grids (grid.py:121-140, geometry.py:97-151): lon/lat and xyz of two
    rotated grids, and the serial O32 -> rotated O16 remap (stencils + apply); mesh_stats /
    total_area of a few serial meshes (mesh.py:355-420)."""
    from spheregrid.geometry import RotationSpec
    from spheregrid.grid import GridKind, GridSpec, build_grid
    from spheregrid.mesh import mesh_stats, total_area
    out = {}
    for tag, kind, n, rot in [("F8", GridKind.FULL_GAUSSIAN, 8, (10.0, 45.0)),
                              ("O16", GridKind.OCTAHEDRAL_GAUSSIAN, 16, (-40.0, 30.0))]:
        g = build_grid(GridSpec(kind, n, projection=RotationSpec(*rot)))
        out[f"{tag}_rot"] = np.array(rot)
        out[f"{tag}_lonlats"] = g.lonlats()
        out[f"{tag}_xyz"] = g.xyz()
    S = R.grid_from_name("O32")
    T = build_grid(GridSpec(GridKind.OCTAHEDRAL_GAUSSIAN, 16, projection=RotationSpec(-40.0, 30.0)))
    dist = R.blocks_partition(S, 1)
    mesh = R.generate_mesh(S, dist, 0, halo=2, include_pole=True)
    fs = R.NodeColumns(mesh, None)
    tdist = R.matching_partition(T, S, dist)
    w = R.build_remap(fs, T, tdist)
    f = fs.create_field("src", levels=3)
    f.host[:] = np.random.default_rng(2026).normal(size=f.host.shape)
    tf = R.StructuredColumns(T, tdist, 0).create_field("dst", levels=3)
    R.apply_remap(w, f, tf)
    for k, v in stencil_arrays(w).items():
        out["remap_" + k] = v
    out["remap_out"] = tf.host
    out["remap_part_of"] = tdist.part_of
    stats = []
    for name, pole, P, part, halo in [("F1", False, 1, 0, 0), ("F1", True, 1, 0, 0), ("O8", True, 1, 0, 0),
                                      ("F8", False, 4, 1, 1), ("O16", True, 3, 2, 2)]:
        g = R.grid_from_name(name)
        m = R.generate_mesh(g, R.blocks_partition(g, P), part, halo=halo, include_pole=pole)
        st = mesh_stats(m)
        stats.append([st[k] for k in ("V", "E", "F", "chi", "owned_nodes", "owned_elements")])
        out[f"area_{name}_{int(pole)}_{P}_{part}_{halo}"] = np.array(total_area(m))
    out["mesh_stats"] = np.array(stats, dtype=np.int64)
    save("rotated", **out)


def _digest(a) -> str:
    import hashlib

    a = np.ascontiguousarray(a)
    return f"{a.dtype.str}:{'x'.join(map(str, a.shape))}:" + hashlib.sha256(a.tobytes()).hexdigest()


def mesh_digest_fields(mesh):
    conn = mesh.element_connectivity
    return {"node_global": _digest(mesh.node_global.astype(np.int64)),
            "node_xyz": _digest(mesh.node_xyz.astype(np.float64)),
            "node_part": _digest(mesh.node_part.astype(np.int32)),
            "node_remote": _digest(mesh.node_remote.astype(np.int64)),
            "node_halo": _digest(mesh.node_halo.astype(np.int16)),
            "node_ghost": _digest(mesh.node_ghost.astype(bool)),
            "conn_offsets": _digest(conn.offsets.astype(np.int64)),
            "conn_indices": _digest(conn.indices.astype(np.int64)),
            "elem_serial_id": _digest(mesh.elem_serial_id.astype(np.int64)),
            "nb_nodes": int(mesh.nb_nodes), "nb_elements": int(mesh.nb_elements)}


def mesh_digests(ranks=(0, 3, 7)):
    """sha256 digests of the O1280 grids (latitudes, lonlats, xyz), the serial O1280 halo-2
    mesh with poles (the cfg3 source) and ranks of the O1280 P=8 halo-2 blocks meshes (the
    N>1 bench): the full arrays are too large to commit, their digests pin them bitwise."""
    import json

    out = {}
    path = os.path.join(HERE, "mesh_digests.json")
    if os.path.exists(path):
        with open(path) as fh:
            out = json.load(fh)

    def dump():
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)
        print("wrote", path, sorted(out), flush=True)

    for name in ("O1280", "O640"):
        G = R.grid_from_name(name)
        out[f"grid_{name}"] = {"latitudes": _digest(G.latitudes), "lonlats": _digest(G.lonlats()),
                               "xyz": _digest(G.xyz()), "npts": int(G.npts)}
    dump()
    S = R.grid_from_name("O1280")
    t = time.time()
    out["mesh_O1280_p1_h2"] = mesh_digest_fields(R.generate_mesh(S, R.blocks_partition(S, 1), 0, halo=2,
                                                                 include_pole=True))
    print("serial mesh", round(time.time() - t, 1), flush=True)
    dump()
    dist = R.blocks_partition(S, 8)
    for r in ranks:
        t = time.time()
        out[f"mesh_O1280_p8_h2_r{r}"] = mesh_digest_fields(R.generate_mesh(S, dist, r, halo=2, include_pole=True))
        print("rank", r, round(time.time() - t, 1), flush=True)
        dump()


DEGENERATE_GRIDS = {
    # a 2-point row puts its points at lon 0 and 180: every triangle it makes with the pole
    # (and the quads between two such rows) lies in the plane y = 0 -> |triple| <= 1e-15
    "polar2": ((60.0, 2), (30.0, 8), (0.0, 8), (-30.0, 8), (-60.0, 3)),
    "mid2": ((70.0, 6), (40.0, 2), (10.0, 8), (-20.0, 12), (-50.0, 5)),
    "two2": ((75.0, 4), (45.0, 2), (15.0, 2), (-15.0, 10), (-45.0, 7), (-75.0, 3)),
}
DEGENERATE_TARGETS = ("O8", "O16", "F12")


def degenerate():
    """MeshLocator.locate (interp.py:102-117) on custom grids whose meshes hold degenerate
    triangles: per target the outcome (0 located, 1 NotLocated, 2 DegenerateTriangle raised
    while constructing a kNN candidate, interp.py:34-43), the element and corners; and for the
    located ones whether barycentric_weights raises (interp.py:61-71)."""
    out = {}
    for gname, rows in DEGENERATE_GRIDS.items():
        S = R.build_grid(R.GridSpec(kind=R.GridKind.CUSTOM, rows=rows))
        mesh = R.generate_mesh(S, R.blocks_partition(S, 1), 0, halo=0, include_pole=True)
        loc = RI.MeshLocator(mesh)
        out[f"{gname}__rows"] = np.array(rows, dtype=np.float64)
        out[f"{gname}__node_xyz"] = mesh.node_xyz
        for tname in DEGENERATE_TARGETS:
            T = R.grid_from_name(tname)
            xyz = T.xyz()
            code = np.zeros(T.npts, np.int8)
            elem = np.full(T.npts, -1, np.int64)
            corners = np.full((T.npts, 3), -1, np.int64)
            wcode = np.zeros(T.npts, np.int8)
            for t in range(T.npts):
                try:
                    e, tri, c = loc.locate(xyz[t])
                except R.errors.NotLocated:
                    code[t] = 1
                    continue
                except R.errors.DegenerateTriangle:
                    code[t] = 2
                    continue
                elem[t], corners[t] = e, c
                try:
                    RI.barycentric_weights(tri, xyz[t])
                except R.errors.DegenerateTriangle:
                    wcode[t] = 1
            key = f"{gname}__{tname}"
            out[key + "__code"], out[key + "__elem"] = code, elem
            out[key + "__corners"], out[key + "__wcode"] = corners, wcode
            print(gname, tname, np.bincount(code, minlength=3), int(wcode.sum()), flush=True)
    save("degenerate", **out)


def gather_scatter():
    """gather_field / scatter_field (functionspace.py:185-224) at P = 1, 2, 4: NodeColumns on
    O32 (mesh halo 1, poles) with seeded owned values -> the gathered global array and every
    rank's message counters; StructuredColumns scatter of a global array -> each rank's rows
    and counters."""
    out = {}
    g = R.grid_from_name("O32")
    for kind, levels in [(R.Kind.REAL64, 4), (R.Kind.INT32, 3)]:
        tag = kind.name.lower()
        rng = np.random.default_rng(91)
        gvals = rng.normal(size=(g.npts + 2, levels)) * 1e3
        gvals = gvals.astype(kind.dtype)
        out[f"{tag}_values"] = gvals
        for P in (1, 2, 4):
            def program(ctx):
                c = ctx if ctx.nranks > 1 else None
                dist = R.blocks_partition(g, ctx.nranks)
                mesh = R.generate_mesh(g, dist, ctx.rank, halo=1, include_pole=True)
                fs = R.NodeColumns(mesh, c)
                f = fs.create_field("n", levels, kind)
                own = fs.owned_row_index()
                f.host[own] = gvals[mesh.node_global[own]]
                m0 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
                gathered = R.gather_field(fs, f, c)
                m1 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
                sfs = R.StructuredColumns(g, dist, ctx.rank)
                sf = sfs.create_field("s", levels, kind)
                R.scatter_field(sfs, sf, c, gvals[: g.npts] if ctx.rank == 0 else None)
                m2 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
                return gathered, np.array([np.subtract(m1, m0), np.subtract(m2, m1)]), sf.host.copy()
            res = R.run_ranks(P, program)
            out[f"{tag}_p{P}_gathered"] = res[0][0]
            for r in range(P):
                out[f"{tag}_p{P}_r{r}_counters"] = res[r][1]
                out[f"{tag}_p{P}_r{r}_scattered"] = res[r][2]
    save("gather_scatter", **out)


JOBS = {
    "rotated": rotated,
    "degenerate": degenerate,
    "gather_scatter": gather_scatter,
    "checksum": checksums,
    "latitudes": latitudes,
    "cfg1": lambda: serial_remap("O32", "O16", 10, "cfg1_O32_O16"),
    "f8": lambda: serial_remap("F8", "F4", 2, "serial_F8_F4"),
    "p4": lambda: partitioned("O32", "O16", 4, 2, "part_O32_O16_p4_h2"),
    "f8p": lambda: partitioned("F8", "F4", 3, 1, "part_F8_F4_p3_h1"),
    "p8": lambda: partitioned("O160", "O80", 8, 3, "part_O160_O80_p8_h3", levels=2),
    "fallback": fallback_case,
    "matching": matching,
    "cfg2": lambda: serial_remap("O320", "O160", 1, "cfg2_O320_O160"),
    "o1280": o1280_sample,
    "digests": mesh_digests,
}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(JOBS):
        JOBS[name]()
