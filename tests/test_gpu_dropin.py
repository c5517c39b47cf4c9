"""Behaviours the reference's own test-suite asserts for the hot path (test_interp.py,
test_field.py, test_acceptance.py), re-expressed against the drop-in package on the GPU."""
import io
import json

import numpy as np
import pytest

import paper_1908_07038_b200 as sg
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def unit(v):
    v = np.asarray(v, float)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def test_random_points_located_on_closed_mesh(gpu):
    """test_interp.py:116-126: 10,000 random points on F8 (poles) are all located in a
    triangle that contains them; the winner equals the oracle's (reference locate order)."""
    g = sg.grid_from_name("F8")
    mesh = sg.generate_mesh(g, sg.blocks_partition(g, 1), 0, include_pole=True)
    loc = sg.MeshLocator(mesh)
    pts = unit(np.random.default_rng(11).normal(size=(10000, 3)))
    elem, corners = loc.locate_many(pts)
    assert (elem >= 0).all()
    conn = mesh.element_connectivity
    oe, oc = O.locate(mesh.node_xyz, conn.offsets, conn.indices, pts)
    assert np.array_equal(elem, oe) and np.array_equal(corners, oc)
    for k in range(0, 10000, 97):
        tri = sg.SphericalTriangle(*mesh.node_xyz[corners[k]])
        assert sg.contains(tri, pts[k])
        assert set(corners[k].tolist()) <= set(conn.row(elem[k]).tolist())


def test_grid_points_land_on_themselves(gpu):
    """test_interp.py:128-140 + exact ties: a target on a mesh node (several triangles tie at
    score 0) resolves like the reference."""
    g = sg.grid_from_name("O4")
    mesh = sg.generate_mesh(g, sg.blocks_partition(g, 1), 0, include_pole=True)
    loc = sg.MeshLocator(mesh)
    conn = mesh.element_connectivity
    pts = mesh.node_xyz
    elem, corners = loc.locate_many(pts)
    oe, oc = O.locate(pts, conn.offsets, conn.indices, pts)
    assert np.array_equal(elem, oe) and np.array_equal(corners, oc)
    for gidx in [0, 5, g.npts // 2, g.npts - 1]:
        _, tri, c = loc.locate(pts[gidx])
        w = sg.barycentric_weights(tri, pts[gidx])
        k = int(np.argmax(w))
        assert c[k] == gidx and abs(w[k] - 1.0) < 1e-12


def test_identity_remap_f4(gpu):
    """test_interp.py:186-194: F4 -> F4 is the identity; every target sits on a node."""
    g = sg.grid_from_name("F4")
    mesh = sg.generate_mesh(g, sg.blocks_partition(g, 1), 0, halo=0, include_pole=True)
    fs = sg.NodeColumns(mesh, None)
    w = sg.build_remap(fs, g, sg.blocks_partition(g, 1))
    ref = O.build_remap(mesh.node_xyz, mesh.element_connectivity.offsets, mesh.element_connectivity.indices,
                        g.xyz())
    assert np.array_equal(w.nodes, ref["nodes"])
    src = fs.create_field("v")
    src.host[:, 0] = np.cos(np.arange(fs.nb_nodes, dtype=float))
    out = sg.create_field("t", (len(w), 1))
    sg.apply_remap(w, src, out)
    assert np.allclose(out.host[:, 0], src.host[w.target_global, 0], atol=1e-12)


def test_not_located_outside_local_patch(gpu):
    """test_interp.py:142-150."""
    g = sg.grid_from_name("F8")
    mesh = sg.generate_mesh(g, sg.blocks_partition(g, 4), 0, halo=0)
    loc = sg.MeshLocator(mesh)
    lam, phi = np.radians(0.0), np.radians(-85.0)
    p = np.array([np.cos(phi) * np.cos(lam), np.cos(phi) * np.sin(lam), np.sin(phi)])
    with pytest.raises(sg.NotLocated):
        loc.locate(p)


def test_not_located_and_fallback_f8_f16(gpu):
    """test_interp.py:196-218, and the reported target index equals the oracle's first."""
    g, tgt = sg.grid_from_name("F8"), sg.grid_from_name("F16")
    dist = sg.blocks_partition(g, 4)
    mesh = sg.generate_mesh(g, dist, 0, halo=0)
    fs = sg.NodeColumns(mesh, None)
    tdist = sg.matching_partition(tgt, g, dist)
    with pytest.raises(sg.NotLocated) as exc:
        sg.build_remap(fs, tgt, tdist)
    owned = np.flatnonzero(tdist.part_of == 0)
    e, _ = O.locate(mesh.node_xyz, mesh.element_connectivity.offsets, mesh.element_connectivity.indices,
                    tgt.xyz()[owned])
    assert exc.value.target_global_index == int(owned[np.argmax(e < 0)])
    assert "halo" in str(exc.value)
    w = sg.build_remap(fs, tgt, tdist, allow_fallback=True)
    assert w.fallback.any() and np.array_equal(w.fallback, e < 0)
    rows = w.weights[w.fallback]
    assert np.allclose(rows[:, 0], 1.0) and np.allclose(rows[:, 1:], 0.0)


def test_export_rows(gpu):
    g, tgt = sg.grid_from_name("O8"), sg.grid_from_name("F2")
    mesh = sg.generate_mesh(g, sg.blocks_partition(g, 1), 0, halo=0, include_pole=True)
    w = sg.build_remap(sg.NodeColumns(mesh, None), tgt, sg.blocks_partition(tgt, 1))
    buf = io.StringIO()
    sg.export_weights(w, buf)
    lines = buf.getvalue().strip().split("\n")
    assert len(lines) == tgt.npts
    row = json.loads(lines[0])
    assert set(row) == {"target_global_index", "source_global_indices", "weights", "fallback"}
    assert abs(sum(row["weights"]) - 1.0) < 1e-12


def test_serial_parallel_equivalence_and_zero_messages(gpu):
    """test_interp.py:265-272 and test_acceptance.py:167-205 (O32 -> F8 on 32 ranks)."""
    serial, exact, _ = sg.run_remap_pipeline("O8", "F4", 1, "harmonic:Y2,0")
    par, exact2, msgs = sg.run_remap_pipeline("O8", "F4", 4, "harmonic:Y2,0")
    assert np.array_equal(exact, exact2)
    assert np.max(np.abs(serial - par)) < 1e-13
    assert sum(msgs) == 0
    got, exact, msgs = sg.run_remap_pipeline("O32", "F8", 32, "constant:1")
    assert sum(msgs) == 0 and np.abs(got - 1.0).max() < 1e-14


TRANSITIONS = {
    "host_only": {"host_read": "host_only", "host_write": "host_only", "device_read": "raised",
                  "device_write": "raised", "update_host": "raised", "update_device": "raised"},
    "synced": {"host_read": "synced", "host_write": "host_dirty", "device_read": "synced",
               "device_write": "device_dirty", "update_host": "synced", "update_device": "synced"},
    "host_dirty": {"host_read": "host_dirty", "host_write": "host_dirty", "device_read": "raised",
                   "device_write": "raised", "update_host": "host_dirty", "update_device": "synced"},
    "device_dirty": {"host_read": "raised", "host_write": "raised", "device_read": "device_dirty",
                     "device_write": "device_dirty", "update_host": "synced", "update_device": "device_dirty"},
}


def _field_in(state):
    f = sg.create_field("t", (2, 1))
    if state == "host_only":
        return f
    f.allocate_device()
    if state == "host_dirty":
        with f.host_view(sg.Intent.READ_WRITE) as a:
            a[:] = 1
    elif state == "device_dirty":
        with f.device_view(sg.Intent.READ_WRITE) as a:
            a[:] = 1
    return f


def _drive(f, op):
    try:
        if op == "host_read":
            with f.host_view(sg.Intent.READ):
                pass
        elif op == "host_write":
            with f.host_view(sg.Intent.READ_WRITE) as a:
                a[:] = a + 1
        elif op == "device_read":
            with f.device_view(sg.Intent.READ):
                pass
        elif op == "device_write":
            with f.device_view(sg.Intent.READ_WRITE) as a:
                a[:] = a + 1
        elif op == "update_host":
            f.update_host()
        elif op == "update_device":
            f.update_device()
    except (sg.StaleHost, sg.StaleDevice, sg.NoDevice):
        return "raised"
    return f.state.value


@pytest.mark.parametrize("state", list(TRANSITIONS))
@pytest.mark.parametrize("op", ["host_read", "host_write", "device_read", "device_write", "update_host",
                                "update_device"])
def test_state_machine_exhaustive_on_hbm(gpu, state, op):
    """test_field.py:181-226 with a real HBM mirror: Synced implies bitwise-equal buffers."""
    f = _field_in(state)
    assert f.state.value == state
    assert _drive(f, op) == TRANSITIONS[state][op]
    if f.state is sg.MemoryState.SYNCED:
        assert f.host.tobytes() == f.device.tobytes()


def test_device_view_numpy_semantics(gpu):
    """test_field.py:82-91, 132-139: element writes through a device view, reads back."""
    f = sg.create_field("t", (2, 3)).allocate_device()
    with f.device_view(sg.Intent.READ_WRITE) as a:
        for i in range(2):
            for j in range(3):
                a[i, j] = (i + 1) * 100 + (j + 1)
    assert f.state is sg.MemoryState.DEVICE_DIRTY
    f.update_host()
    assert f.host.ravel().tolist() == [101, 102, 103, 201, 202, 203]
    with f.host_view(sg.Intent.READ_WRITE) as a:
        a[:] = 3
    f.update_device()
    assert np.all(f.device == 3) and f.copy_counters["host_to_device"] == 2
    before = dict(f.copy_counters)
    with f.host_view(sg.Intent.READ):
        pass
    with f.device_view(sg.Intent.READ) as d:
        assert np.array_equal(d, np.full((2, 3), 3.0))
    assert f.copy_counters == before


@pytest.mark.parametrize("P", [4, 8])
def test_equal_regions_pipeline_and_halo(gpu, P):
    """Equal-regions partitions (many neighbours per rank): halo ghosts equal their global ids,
    the distributed remap equals the serial one, stencils equal the scaled oracle's."""
    g = sg.grid_from_name("O64")
    d = sg.equal_regions_partition(g, P)

    def prog(ctx):
        mesh = sg.generate_mesh(g, d, ctx.rank, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        f = fs.create_field("g", 2, sg.Kind.INT64)
        own = fs.owned_row_index()
        f.host[own] = mesh.node_global[own, None]
        fs.halo_exchange(f, ctx)
        t = sg.grid_from_name("O32")
        w = sg.build_remap(fs, t, sg.matching_partition(t, g, d))
        conn = mesh.element_connectivity
        e, c = O.locate_kdtree(mesh.node_xyz, conn.offsets, conn.indices, t.xyz()[w.target_global])
        return (np.array_equal(f.host, np.repeat(mesh.node_global[:, None], 2, axis=1)),
                len(fs.exchange_plan.peers), bool((e >= 0).all() and np.array_equal(c, w.nodes)))

    res = sg.run_ranks(P, prog)
    assert all(r[0] and r[2] for r in res)
    serial, _, _ = sg.run_remap_pipeline("O64", "O32", 1, "harmonic:Y3,1")
    par, _, msgs = sg.run_remap_pipeline("O64", "O32", P, "harmonic:Y3,1", partitioner="equal_regions")
    assert np.max(np.abs(serial - par)) < 1e-13 and sum(msgs) == 0


def test_custom_grid_remap_vs_oracle(gpu):
    """A custom row grid (GridSpec CUSTOM, grid.py:28-40) as the source: mesh, stencils and
    apply follow the same code path; stencils equal the reference algorithm's."""
    lats = np.linspace(80.0, -80.0, 17)
    rows = tuple((float(la), int(12 + 4 * (8 - abs(k - 8)))) for k, la in enumerate(lats))
    S = sg.build_grid(sg.GridSpec(kind=sg.GridKind.CUSTOM, rows=rows))
    T = sg.grid_from_name("F6")
    dist = sg.blocks_partition(S, 1)
    mesh = sg.generate_mesh(S, dist, 0, halo=0, include_pole=True)
    w = sg.build_remap(sg.NodeColumns(mesh, None), T, sg.matching_partition(T, S, dist), allow_fallback=True)
    conn = mesh.element_connectivity
    e, c = O.locate_kdtree(mesh.node_xyz, conn.offsets, conn.indices, T.xyz())
    assert np.array_equal(e < 0, w.fallback)
    assert np.array_equal(w.nodes[~w.fallback], c[~w.fallback])


def test_cli_remap_report(gpu, tmp_path):
    """test_cli.py:132-152: the remap subcommand's report and dump format."""
    import subprocess
    import sys

    from conftest import ROOT

    out = tmp_path / "f.txt"
    r = subprocess.run([sys.executable, "-m", "paper_1908_07038_b200", "remap", "--source", "O8", "--target", "F4",
                        "--parts", "2", "--field", "constant:1", "--out", str(out), "--report"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    report = dict(line.split(": ") for line in r.stdout.strip().splitlines() if ": " in line)
    assert float(report["max_error"]) < 1e-13
    assert int(report["messages_during_interpolation"]) == 0
    text = out.read_text()
    assert text.startswith("# field:")
    assert len([ln for ln in text.splitlines() if not ln.startswith("#")]) == 128


def test_integration_dropin_snippet_runs(gpu):
    """INTEGRATION.md's drop-in program (the reference pipeline's order, cli.py:119-154) runs as
    written on this package — grid names shrunk to O32 -> O16 so it takes seconds; 8 ranks
    on the test box's GPU."""
    import os
    import re

    from conftest import ROOT

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(.*?)```", text, re.S).group(1)
    code = "\n".join(line[3:] if line.startswith("   ") else line for line in block.splitlines())
    assert '"O1280"' in code and '"O640"' in code and "sg.run_ranks(8, program)" in code
    code = code.replace('"O1280"', '"O32"').replace('"O640"', '"O16"')
    code = code.replace("sg.apply_remap(w, f, tf)", "sg.apply_remap(w, f, tf)\n    return len(w), tf.host.shape")
    code = code.replace("sg.run_ranks(8, program)", "RESULT = sg.run_ranks(8, program)")
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    assert sum(r[0] for r in ns["RESULT"]) == sg.grid_from_name("O16").npts
    assert all(r[1][1] == 137 for r in ns["RESULT"])
