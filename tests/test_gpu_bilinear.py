"""Structured-bilinear remap (BASELINE configs[4]).  The reference has no bilinear method,
so parity is against the repo's own CPU restatement (oracle.bilinear_stencil) — "parity
unpinned" vs the reference — plus analytic properties."""
import numpy as np
import pytest

import paper_1908_07038_b200 as sg
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_bilinear_serial_bitwise_vs_restatement(gpu):
    S, T = sg.grid_from_name("O64"), sg.grid_from_name("O32")
    dist = sg.blocks_partition(S, 1)
    mesh = sg.generate_mesh(S, dist, 0, halo=0, include_pole=True)
    fs = sg.NodeColumns(mesh, None)
    td = sg.matching_partition(T, S, dist)
    w = sg.build_bilinear(fs, T, td)
    gn, ww, ok = O.bilinear_stencil(S.latitudes, S.nlons, T.lonlats(), True)
    assert ok.all()
    assert np.array_equal(mesh.node_global[w.nodes], gn)
    assert np.array_equal(w.weights.view(np.uint64), ww.view(np.uint64))
    assert np.abs(w.weights.sum(1) - 1).max() < 1e-14
    h = np.random.default_rng(4).normal(size=(mesh.nb_nodes, 137))
    f = fs.create_field("s", 137)
    f.host[:] = h
    tf = sg.StructuredColumns(T, td, 0).create_field("t", 137)
    sg.apply_remap(w, f, tf)
    exp = O.apply_remap_k(w.nodes, w.weights, h)
    assert np.array_equal(tf.host.view(np.uint64), exp.view(np.uint64))


def test_bilinear_caps_and_no_poles(gpu):
    # a finer target than the source reaches into the polar caps
    S, T = sg.grid_from_name("O16"), sg.grid_from_name("O64")
    dist = sg.blocks_partition(S, 1)
    mesh = sg.generate_mesh(S, dist, 0, halo=0, include_pole=True)
    td = sg.matching_partition(T, S, dist)
    w = sg.build_bilinear(sg.NodeColumns(mesh, None), T, td)
    gn, ww, ok = O.bilinear_stencil(S.latitudes, S.nlons, T.lonlats(), True)
    assert np.array_equal(mesh.node_global[w.nodes], gn)
    assert np.array_equal(w.weights.view(np.uint64), ww.view(np.uint64))
    const = np.full((mesh.nb_nodes, 1), 2.5)
    assert np.abs(O.apply_remap_k(w.nodes, w.weights, const) - 2.5).max() < 1e-14
    mesh0 = sg.generate_mesh(S, dist, 0, halo=0, include_pole=False)
    with pytest.raises(sg.NotLocated):
        sg.build_bilinear(sg.NodeColumns(mesh0, None), T, td)


@pytest.mark.parametrize("P,halo", [(4, 1), (4, 2), (8, 2)])
def test_bilinear_partitioned_matches_serial(gpu, P, halo):
    S, T = sg.grid_from_name("O64"), sg.grid_from_name("O32")
    gn, ww, _ = O.bilinear_stencil(S.latitudes, S.nlons, T.lonlats(), True)
    dist = sg.blocks_partition(S, P)
    td = sg.matching_partition(T, S, dist)
    for r in range(P):
        mesh = sg.generate_mesh(S, dist, r, halo=halo, include_pole=True)
        w = sg.build_bilinear(sg.NodeColumns(mesh, None), T, td)
        assert np.array_equal(mesh.node_global[w.nodes], gn[w.target_global])
        assert np.array_equal(w.weights, ww[w.target_global])


def test_bilinear_second_order(gpu):
    """Y_2^0 error shrinks ~4x per resolution doubling (bilinear is second order)."""
    spec = sg.FieldSpec("harmonic:Y2,0")
    errs = []
    for sname, tname in (("O32", "O24"), ("O64", "O48")):
        S, T = sg.grid_from_name(sname), sg.grid_from_name(tname)
        dist = sg.blocks_partition(S, 1)
        mesh = sg.generate_mesh(S, dist, 0, halo=0, include_pole=True)
        fs = sg.NodeColumns(mesh, None)
        td = sg.matching_partition(T, S, dist)
        interp = sg.Interpolation(fs, T, td, method="structured-bilinear")
        f = fs.create_field("s", 1)
        f.host[:, 0] = spec(mesh.node_xyz)
        tf = sg.StructuredColumns(T, td, 0).create_field("t", 1)
        interp.execute(f, tf)
        errs.append(np.abs(tf.host[:, 0] - spec(T.xyz())).max())
    assert 2.5 < errs[0] / errs[1] < 6
