"""Host-side prerequisites of the hot path (grid, latitudes, partitions, per-partition
mesh numbering — native C++ for the integer parts) are bit-identical to the reference's
golden fixtures.  CPU only."""
import numpy as np
import pytest

import paper_1908_07038_b200 as sg


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32, 64, 80, 160, 320, 640, 1280])
def test_gaussian_latitudes_bitwise(golden, n):
    z = golden("latitudes")
    assert np.array_equal(sg.gaussian_latitudes(n).view(np.uint64), z[f"n{n}"].view(np.uint64))


def test_grid_numerology():
    assert sg.grid_from_name("F8").npts == 512
    assert sg.grid_from_name("O32").npts == 5248
    assert sg.grid_from_name("O1280").npts == 6599680
    with pytest.raises(sg.UnknownGridName):
        sg.grid_from_name("bogus")


def test_f1_point_latitude():
    # test_cli.py:84-88 known answer
    assert sg.grid_from_name("F1").latitudes[1] == -35.264389682754654


@pytest.mark.parametrize("name", ["part_O32_O16_p4_h2", "part_F8_F4_p3_h1", "part_O160_O80_p8_h3"])
def test_partition_meshes_bitwise(golden, name):
    z = golden(name)
    sname = {"part_O32_O16_p4_h2": "O32", "part_F8_F4_p3_h1": "F8", "part_O160_O80_p8_h3": "O160"}[name]
    S = sg.grid_with_latitudes(sname, z["src_lat"])
    P, halo = int(z["nparts"]), int(z["halo"])
    dist = sg.blocks_partition(S, P)
    for r in range(P):
        m = sg.generate_mesh(S, dist, r, halo=halo, include_pole=True)
        for k in ["node_global", "node_part", "node_remote", "node_halo"]:
            assert np.array_equal(getattr(m, k), z[f"r{r}_{k}"]), (r, k)
        assert np.array_equal(m.element_connectivity.offsets, z[f"r{r}_conn_off"])
        assert np.array_equal(m.element_connectivity.indices, z[f"r{r}_conn_idx"])
        assert np.array_equal(m.elem_serial_id, z[f"r{r}_elem_serial"])


@pytest.mark.parametrize("tgt,src,P", [("O16", "O32", 4), ("O80", "O160", 8), ("O160", "O320", 8),
                                       ("O640", "O1280", 8)])
def test_matching_partition_bitwise(golden, tgt, src, P):
    z = golden("matching")
    S, T = sg.grid_from_name(src), sg.grid_from_name(tgt)
    idx = sg.partition.nearest_master_points(S, T.xyz())
    assert np.array_equal(idx, z[f"{tgt}_{src}_idx"])
    d = sg.matching_partition(T, S, sg.blocks_partition(S, P))
    assert np.array_equal(d.part_of, z[f"{tgt}_{src}_p{P}"])


def test_blocks_partition_sizes():
    g = sg.grid_from_name("O32")
    d = sg.blocks_partition(g, 3)
    assert d.counts.tolist() == [1750, 1749, 1749]
    assert np.all(np.diff(d.part_of) >= 0)
    with pytest.raises(sg.TooManyParts):
        sg.blocks_partition(sg.grid_from_name("F1"), 100)


def test_serial_mesh_counts():
    # element counts of the serial meshes with poles
    for name, ne in [("O32", 10104), ("O320", 838392)]:
        g = sg.grid_from_name(name)
        m = sg.generate_mesh(g, sg.blocks_partition(g, 1), 0, halo=0, include_pole=True)
        assert m.nb_elements == ne
        assert m.nb_nodes == g.npts + 2


def test_split_quad_lowest_local_index():
    tri = sg.split_quad(np.array([7, 3, 9, 5]))
    assert [t.tolist() for t in tri] == [[3, 9, 5], [3, 5, 7]]


def test_dump_field_format():
    """field.py:190-202 format (the reference's own expected layout, test_field.py:250)."""
    import io

    f = sg.create_field("t", (2, 2))
    f.host[:] = [[1.5, 2.0], [1e-300, -3.25]]
    buf = io.StringIO()
    sg.dump_field(f, np.array([7, 9]), buf)
    assert buf.getvalue().splitlines() == ["# field: t", "# shape: 2 2", "# kind: real64", "7 0 1.5", "7 1 2",
                                           "9 0 1e-300", "9 1 -3.25"]


def test_distribution_to_dict():
    d = sg.blocks_partition(sg.grid_from_name("F1"), 2)
    assert d.to_dict() == {"nparts": 2, "counts": [4, 4], "part_of": [0, 0, 0, 0, 1, 1, 1, 1]}


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8, 16, 32])
def test_equal_regions_balanced_and_compact(P):
    """Equal-regions decomposition (extension; the reference has only blocks): part sizes equal
    blocks_partition's, every part is a compact region (fewer ghosts than bands at P >= 4)."""
    from paper_1908_07038_b200.partition import eq_regions_collars

    g = sg.grid_from_name("O64")
    d = sg.equal_regions_partition(g, P)
    assert sum(eq_regions_collars(P)) == P
    assert d.counts.tolist() == sg.blocks_partition(g, P).counts.tolist()
    assert np.array_equal(d.part_of, sg.equal_regions_partition(g, P).part_of)  # deterministic
    if P >= 4:
        def ghosts(dist):
            return sum(int(sg.generate_mesh(g, dist, r, halo=2, include_pole=True).node_ghost.sum())
                       for r in range(P))
        assert ghosts(d) < ghosts(sg.blocks_partition(g, P))


def test_grid_point_and_geometry_helpers():
    """grid_point (grid.py:128-135), PointLonLat / lonlat_to_xyz round trip (geometry.py)."""
    g = sg.grid_from_name("O4")
    p = sg.grid_point(g, 5)
    assert p.lat == g.latitudes[0] and p.lon == 360.0 * 5 / 20
    v = sg.lonlat_to_xyz(sg.PointLonLat(-30.0, 45.0))
    q = sg.xyz_to_lonlat(v)
    assert abs(q.lon - 330.0) < 1e-12 and abs(q.lat - 45.0) < 1e-12
    with pytest.raises(sg.NotOnUnitSphere):
        sg.PointXYZ(1.0, 1.0, 0.0)
    assert g.describe()["npts"] == g.npts


def _rotated_grid(tag, z):
    from paper_1908_07038_b200.grid import GridKind, GridSpec, build_grid
    kind = GridKind.FULL_GAUSSIAN if tag.startswith("F") else GridKind.OCTAHEDRAL_GAUSSIAN
    return build_grid(GridSpec(kind, int(tag[1:]), projection=sg.RotationSpec(*z[f"{tag}_rot"])))


@pytest.mark.parametrize("tag", ["F8", "O16"])
def test_rotated_grid_coordinates_equal_reference(golden, tag):
    """grid.py:121-140: rotated lon/lat and xyz bit-identical to the reference's."""
    z = golden("rotated")
    g = _rotated_grid(tag, z)
    assert np.array_equal(g.lonlats().view(np.uint64), z[f"{tag}_lonlats"].view(np.uint64))
    assert np.array_equal(g.xyz().view(np.uint64), z[f"{tag}_xyz"].view(np.uint64))
    # scalar path (Grid.point -> unrotate) agrees with the vectorised one to rounding
    for gi in (0, 5, g.npts // 2, g.npts - 1):
        p = g.point(gi)
        lon, lat = z[f"{tag}_lonlats"][gi]
        assert abs(p.lat - lat) < 1e-9 and min(abs(p.lon - lon), 360 - abs(p.lon - lon)) < 1e-9


def test_rotation_round_trip_and_distance():
    r = sg.RotationSpec(10.0, 45.0)
    p = sg.PointLonLat(33.0, -12.5)
    q = sg.unrotate(sg.rotate(p, r), r)
    assert abs(q.lon - p.lon) < 1e-12 and abs(q.lat - p.lat) < 1e-12
    pole = sg.rotate(sg.PointLonLat(10.0, 45.0), r)
    assert abs(pole.lat - 90.0) < 1e-9
    assert sg.rotate(p, sg.RotationSpec()) is p
    a, b = sg.PointLonLat(0.0, 0.0), sg.PointLonLat(90.0, 0.0)
    assert abs(sg.great_circle_distance(a, b) - np.pi / 2) < 1e-15
    # distances are invariant under the rotation
    g0, g1 = sg.PointLonLat(12.0, 40.0), sg.PointLonLat(-70.0, -3.0)
    d0 = sg.great_circle_distance(g0, g1)
    assert abs(sg.great_circle_distance(sg.rotate(g0, r), sg.rotate(g1, r)) - d0) < 1e-12


def test_mesh_stats_and_area_equal_reference(golden):
    """mesh.py:355-420: V/E/F/chi/owned counts exact; L'Huilier area within 1e-12 relative."""
    z = golden("rotated")
    cases = [("F1", False, 1, 0, 0), ("F1", True, 1, 0, 0), ("O8", True, 1, 0, 0), ("F8", False, 4, 1, 1),
             ("O16", True, 3, 2, 2)]
    for row, (name, pole, P, part, halo) in zip(z["mesh_stats"], cases):
        g = sg.grid_from_name(name)
        m = sg.generate_mesh(g, sg.blocks_partition(g, P), part, halo=halo, include_pole=pole)
        st = sg.mesh_stats(m)
        assert [st[k] for k in ("V", "E", "F", "chi", "owned_nodes", "owned_elements")] == row.tolist()
        ref = float(z[f"area_{name}_{int(pole)}_{P}_{part}_{halo}"])
        assert abs(sg.total_area(m) - ref) <= 1e-12 * ref


def test_serial_topology_is_global_sweep():
    g = sg.grid_from_name("O2")
    topo = sg.serial_topology(g, include_pole=True)
    m = sg.generate_mesh(g, sg.blocks_partition(g, 1), 0, halo=0, include_pole=True)
    assert topo.nnodes == g.npts + 2 and topo.north_pole == g.npts and topo.south_pole == g.npts + 1
    assert len(topo.elem_nodes) == m.nb_elements
    assert sum(len(e) for e in topo.elem_nodes) == len(m.element_connectivity.indices)
    assert topo.node_lonlat.shape == (g.npts + 2, 2)


def test_runtime_initialise_finalise(monkeypatch):
    """initialise / finalise (runtime.py of the reference): DoubleInitialise on a second
    initialise, the debug channel from SPHEREGRID_DEBUG, warning/error on the error stream."""
    import io

    monkeypatch.setenv("SPHEREGRID_DEBUG", "1")
    out, err = io.StringIO(), io.StringIO()
    lib = sg.initialise(out=out, err=err)
    try:
        with pytest.raises(sg.DoubleInitialise):
            sg.initialise()
        assert lib.config.debug and "debug: version" in out.getvalue()
        lib.log.warning("w")
        lib.log.info("i")
        assert "warning: w" in err.getvalue() and "info: i" in out.getvalue()
    finally:
        sg.finalise()
    sg.finalise()  # idempotent
    monkeypatch.setenv("SPHEREGRID_DEBUG", "0")
    lib = sg.initialise(out=io.StringIO())
    assert not lib.config.debug
    sg.finalise()
