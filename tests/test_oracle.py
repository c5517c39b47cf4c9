"""Pins the oracle (oracle/, the CPU restatement used as the checker) against the golden
fixtures produced by the unmodified reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import paper_1908_07038_b200 as sg
from oracle import oracle as O


def serial_mesh(z, sname):
    S = sg.grid_with_latitudes(sname, z["src_lat"])
    return S, sg.generate_mesh(S, sg.blocks_partition(S, 1), 0, halo=2, include_pole=True)


@pytest.mark.parametrize("name,src,tgt", [("cfg1_O32_O16", "O32", "O16"), ("serial_F8_F4", "F8", "F4")])
def test_oracle_stencils_weights_apply_equal_reference(golden, name, src, tgt):
    z = golden(name)
    S, mesh = serial_mesh(z, src)
    T = sg.grid_with_latitudes(tgt, z["tgt_lat"])
    conn = mesh.element_connectivity
    r = O.build_remap(mesh.node_xyz, conn.offsets, conn.indices, T.xyz()[z["target_global"]])
    assert np.array_equal(r["nodes"], z["nodes"])
    # same LAPACK on the same host: weights and scale are bit-identical to the reference
    assert np.array_equal(r["weights"].view(np.uint64), z["weights"].view(np.uint64))
    assert np.array_equal(r["scale"].view(np.uint64), z["scale"].view(np.uint64))
    src_field = np.random.default_rng(2026).normal(size=(mesh.nb_nodes, z["out"].shape[1]))
    out = O.apply_remap(z["nodes"].astype(np.int64), z["weights"], src_field)
    assert np.array_equal(out.view(np.uint64), z["out"].view(np.uint64))


def test_oracle_partitioned_stencils_equal_reference(golden):
    z = golden("part_O32_O16_p4_h2")
    S = sg.grid_with_latitudes("O32", z["src_lat"])
    T = sg.grid_with_latitudes("O16", z["tgt_lat"])
    P = int(z["nparts"])
    dist = sg.blocks_partition(S, P)
    for r in range(P):
        mesh = sg.generate_mesh(S, dist, r, halo=int(z["halo"]), include_pole=True)
        conn = mesh.element_connectivity
        res = O.build_remap(mesh.node_xyz, conn.offsets, conn.indices, T.xyz()[z[f"r{r}_w_target_global"]])
        assert np.array_equal(res["nodes"], z[f"r{r}_w_nodes"])
        assert np.array_equal(res["weights"].view(np.uint64), z[f"r{r}_w_weights"].view(np.uint64))


def test_oracle_not_located_on_halo_zero(golden):
    z = golden("fallback_O32_O16_p4_h0")
    S, T = sg.grid_from_name("O32"), sg.grid_from_name("O16")
    dist = sg.blocks_partition(S, 4)
    tdist = sg.matching_partition(T, S, dist)
    for r in range(4):
        mesh = sg.generate_mesh(S, dist, r, halo=0, include_pole=True)
        owned = np.flatnonzero(tdist.part_of == r)
        conn = mesh.element_connectivity
        elem, _ = O.locate(mesh.node_xyz, conn.offsets, conn.indices, T.xyz()[owned])
        bad = owned[elem < 0]
        assert (bad[0] if len(bad) else -1) == int(z[f"r{r}_bad"])
        assert np.array_equal(elem < 0, z[f"r{r}_fallback"])


def test_oracle_halo_payloads_equal_reference_bytes(golden):
    z = golden("part_O32_O16_p4_h2")
    P = int(z["nparts"])
    for r in range(P):
        send = {p: z[f"r{r}_send_{p}"] for p in range(P) if f"r{r}_send_{p}" in z.files}
        pay = O.halo_payloads(send, z[f"r{r}_before"])
        for p, b in pay.items():
            assert b == z[f"payload_{r}_{p}"].tobytes()
    for r in range(P):
        recv = {p: z[f"r{r}_recv_{p}"] for p in range(P) if f"r{r}_recv_{p}" in z.files}
        pays = {p: z[f"payload_{p}_{r}"].tobytes() for p in recv}
        out = O.halo_unpack(recv, z[f"r{r}_before"], pays)
        assert np.array_equal(out.view(np.uint64), z[f"r{r}_after"].view(np.uint64))


def test_oracle_matching_equals_reference(golden):
    z = golden("matching")
    S, T = sg.grid_from_name("O32"), sg.grid_from_name("O16")
    assert np.array_equal(O.nearest_points(S.xyz(), T.xyz()), z["O16_O32_idx"])
    # every 16th O80 target against O160 (the brute force is O(n*m))
    S, T = sg.grid_from_name("O160"), sg.grid_from_name("O80")
    sel = np.arange(0, T.npts, 16)
    assert np.array_equal(O.nearest_points(S.xyz(), T.xyz()[sel]), z["O80_O160_idx"][sel])


@pytest.mark.parametrize("n", [1, 2, 8, 16, 32])
def test_oracle_gaussian_latitudes_equal_reference(golden, n):
    z = golden("latitudes")
    assert np.array_equal(O.gaussian_latitudes(n).view(np.uint64), z[f"n{n}"].view(np.uint64))


def test_oracle_blocks_partition():
    assert np.array_equal(O.blocks_partition(10, 3), sg.blocks_partition(sg.grid_from_name("F1"), 3).part_of[:0]
                          if False else np.array([0, 0, 0, 0, 1, 1, 1, 2, 2, 2], np.int32))


@pytest.mark.parametrize("name,src,tgt", [("cfg1_O32_O16", "O32", "O16"), ("cfg2_O320_O160", "O320", "O160")])
def test_oracle_kdtree_locate_equals_reference(golden, name, src, tgt):
    """The scaled oracle (scipy cKDTree candidates + C scoring) reproduces the reference's
    full stencils (cfg2: 108,160 targets)."""
    z = golden(name)
    S, mesh = serial_mesh(z, src)
    T = sg.grid_with_latitudes(tgt, z["tgt_lat"])
    conn = mesh.element_connectivity
    elem, corners = O.locate_kdtree(mesh.node_xyz, conn.offsets, conn.indices, T.xyz()[z["target_global"]])
    assert (elem >= 0).all()
    assert np.array_equal(corners, z["nodes"])
    w = O.barycentric_weights_batched(mesh.node_xyz, corners, T.xyz()[z["target_global"]])
    assert np.abs(w - z["weights"]).max() < 1e-14


def test_bilinear_restatement_properties():
    """The structured-bilinear definition (no reference counterpart): weights form a partition
    of unity, stencil nodes lie in the bracketing rows, and a grid remapped onto itself is the
    identity to rounding (every target sits on a node)."""
    S = sg.grid_from_name("O32")
    gn, w, ok = O.bilinear_stencil(S.latitudes, S.nlons, S.lonlats(), True)
    assert ok.all()
    assert np.abs(w.sum(axis=1) - 1.0).max() < 1e-15
    vals = np.random.default_rng(0).normal(size=(S.npts + 2, 2))
    out = O.apply_remap_k(gn, w, vals)
    assert np.abs(out - vals[: S.npts]).max() < 1e-12  # alpha = (360 i / n) n / 360 - i is 0 up to rounding
    T = sg.grid_from_name("F8")
    gn, w, ok = O.bilinear_stencil(S.latitudes, S.nlons, T.lonlats(), True)
    rows = np.searchsorted(S.row_offset, gn, side="right") - 1
    assert (np.abs(rows[:, 2] - rows[:, 0]) <= 1).all()


def test_oracle_checksum_equals_reference(golden):
    z = golden("checksum")
    for name in ("O32", "F8", "O16"):
        vals = z[f"{name}_values"]
        assert O.checksum_partial(np.arange(len(vals)), vals) == int(z[f"{name}_p1"][0])


def test_oracle_rotated_target_equals_reference(golden):
    """O32 -> rotated O16 (RotationSpec(-40, 30)): the oracle's stencils/weights/apply equal
    the reference's on targets whose coordinates come from the rotated grid."""
    from paper_1908_07038_b200.grid import GridKind, GridSpec, build_grid
    z = golden("rotated")
    S = sg.grid_from_name("O32")
    T = build_grid(GridSpec(GridKind.OCTAHEDRAL_GAUSSIAN, 16, projection=sg.RotationSpec(*z["O16_rot"])))
    mesh = sg.generate_mesh(S, sg.blocks_partition(S, 1), 0, halo=2, include_pole=True)
    conn = mesh.element_connectivity
    r = O.build_remap(mesh.node_xyz, conn.offsets, conn.indices, T.xyz()[z["remap_target_global"]])
    assert np.array_equal(r["nodes"], z["remap_nodes"])
    assert np.array_equal(r["weights"].view(np.uint64), z["remap_weights"].view(np.uint64))
    src = np.random.default_rng(2026).normal(size=(mesh.nb_nodes, 3))
    out = O.apply_remap(z["remap_nodes"].astype(np.int64), z["remap_weights"], src)
    assert np.array_equal(out.view(np.uint64), z["remap_out"].view(np.uint64))


@pytest.mark.parametrize("gname", ["polar2", "mid2", "two2"])
def test_oracle_degenerate_candidates_equal_reference(golden, gname):
    """The oracle's brute-force kNN locate raises DegenerateTriangle (-2) exactly where the
    reference does on meshes with degenerate triangles (interp.py:34-43, 90-117), except at
    exact distance ties at the k-th nearest node (cKDTree order, unpinned)."""
    z = golden("degenerate")
    rows = tuple((float(a), int(b)) for a, b in z[f"{gname}__rows"].tolist())
    S = sg.build_grid(sg.GridSpec(kind=sg.GridKind.CUSTOM, rows=rows))
    mesh = sg.generate_mesh(S, sg.blocks_partition(S, 1), 0, halo=0, include_pole=True)
    assert np.array_equal(mesh.node_xyz.view(np.uint64), z[f"{gname}__node_xyz"].view(np.uint64))
    conn = mesh.element_connectivity
    for tname in ("O8", "O16", "F12"):
        xyz = sg.grid_from_name(tname).xyz()
        elem, _ = O.locate(mesh.node_xyz, conn.offsets, conn.indices, xyz)
        code = np.where(elem >= 0, 0, np.where(elem == -2, 2, 1))
        ref = z[f"{gname}__{tname}__code"]
        diff = np.flatnonzero((code != ref) | ((code == 0) & (elem != z[f"{gname}__{tname}__elem"])))
        assert len(diff) <= 2, (tname, diff)


@pytest.mark.parametrize("name,src,tgt", [("cfg1_O32_O16", "O32", "O16"), ("serial_F8_F4", "F8", "F4"),
                                          ("cfg2_O320_O160", "O320", "O160")])
def test_dgesv_restatement_equals_numpy_and_reference(golden, name, src, tgt):
    """The restated 3x3 dgesv (what csrc/locate.cu computes) equals np.linalg.solve on this
    host and, renormalised, the reference's golden weights, bit for bit (interp.py:61-71)."""
    z = golden(name)
    S, mesh = serial_mesh(z, src)
    T = sg.grid_with_latitudes(tgt, z["tgt_lat"])
    xyz = mesh.node_xyz
    nodes = z["nodes"].astype(np.int64)
    M = np.stack([xyz[nodes[:, 0]], xyz[nodes[:, 1]], xyz[nodes[:, 2]]], axis=2)
    p = T.xyz()[z["target_global"]]
    x = O.dgesv3_restated(M, p)
    ref = np.linalg.solve(M, p[..., None])[..., 0]
    assert np.array_equal(x.view(np.uint64), ref.view(np.uint64))
    s = (x[:, 0] + x[:, 1]) + x[:, 2]
    assert np.array_equal((x / s[:, None]).view(np.uint64), z["weights"].view(np.uint64))
