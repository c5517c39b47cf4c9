"""DegenerateTriangle parity: the reference raises while constructing
ANY candidate triangle of a target's k nearest nodes whose triple product is <= 1e-15
(interp.py:34-43, evaluated at interp.py:109-110), k = 8 then min(32, n) (interp.py:90-117).
Custom grids with 2-point rows put whole elements in the plane y = 0; the fixture
(tests/golden/degenerate.npz, make_golden.py `degenerate`) holds the unmodified reference's
outcome for every target of O8 / O16 / F12 on three such meshes.  The device decides these
meshes with the exact kNN-candidate emulation of locate.cu (knn_rule_kernel); the only
allowed differences are targets with an exact distance tie at the k-th nearest node, where
cKDTree's order is unspecified (parity unpinned there)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRIDS = ("polar2", "mid2", "two2")
TARGETS = ("O8", "O16", "F12")


def _mesh(sg, z, gname):
    rows = tuple((float(a), int(b)) for a, b in z[f"{gname}__rows"].tolist())
    S = sg.build_grid(sg.GridSpec(kind=sg.GridKind.CUSTOM, rows=rows))
    mesh = sg.generate_mesh(S, sg.blocks_partition(S, 1), 0, halo=0, include_pole=True)
    assert np.array_equal(mesh.node_xyz.view(np.uint64), z[f"{gname}__node_xyz"].view(np.uint64))
    return S, mesh


def _tied_at_k(node_xyz, p):
    """Exact squared-distance tie between the k-th and (k+1)-th nearest node, k = 8 or 32."""
    d = node_xyz - p
    d2 = np.sort((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
    kmax = min(32, len(d2))
    return any(k < len(d2) and d2[k - 1] == d2[k] for k in (min(8, kmax), kmax))


@pytest.mark.parametrize("gname", GRIDS)
@pytest.mark.parametrize("tname", TARGETS)
def test_locate_outcomes_equal_reference(gpu, golden, gname, tname):
    sg = gpu
    z = golden("degenerate")
    _, mesh = _mesh(sg, z, gname)
    T = sg.grid_from_name(tname)
    xyz = T.xyz()
    key = f"{gname}__{tname}"
    ref_code, ref_elem, ref_corners = z[key + "__code"], z[key + "__elem"], z[key + "__corners"]
    elem, corners = sg.MeshLocator(mesh).locate_many(xyz)
    assert not (elem == -3).any()
    code = np.where(elem >= 0, 0, np.where(elem == -2, 2, 1))
    assert (ref_code == 2).any() and (ref_code == 0).any()  # the case is exercised both ways
    diff = np.flatnonzero((code != ref_code) | ((code == 0) & (elem != ref_elem)))
    assert all(_tied_at_k(mesh.node_xyz, xyz[t]) for t in diff), [int(t) for t in diff if not
                                                                  _tied_at_k(mesh.node_xyz, xyz[t])]
    assert len(diff) <= 2
    ok = (code == 0) & (ref_code == 0)
    assert np.array_equal(corners[ok], ref_corners[ok])


@pytest.mark.parametrize("gname", GRIDS)
def test_build_remap_raises_like_reference(gpu, golden, gname):
    """build_remap raises the reference's exception class for the first failing target in
    ascending order (interp.py:175-185), DegenerateTriangle even with allow_fallback."""
    sg = gpu
    z = golden("degenerate")
    S, mesh = _mesh(sg, z, gname)
    T = sg.grid_from_name("O16")
    fs = sg.NodeColumns(mesh, None)
    td = sg.matching_partition(T, S, sg.blocks_partition(S, 1))
    ref_code = z[f"{gname}__O16__code"]
    first = int(np.flatnonzero(ref_code != 0)[0])
    assert ref_code[first] == 2
    for fb in (False, True):
        with pytest.raises(sg.DegenerateTriangle):
            sg.build_remap(fs, T, td, None, allow_fallback=fb)
    # the Atlas-style single-point locate raises the same class
    with pytest.raises(sg.DegenerateTriangle):
        sg.MeshLocator(mesh).locate(T.xyz()[first])


def test_meshes_without_degenerate_triangles_keep_the_fast_path(gpu, golden):
    """A regular Gaussian mesh has no degenerate triangle: no target is decided by the kNN
    emulation and the located set equals the golden cfg1 stencils (bit-exact elsewhere)."""
    sg = gpu
    z = golden("cfg1_O32_O16")
    S, T = sg.grid_with_latitudes("O32", z["src_lat"]), sg.grid_with_latitudes("O16", z["tgt_lat"])
    mesh = sg.generate_mesh(S, sg.blocks_partition(S, 1), 0, halo=2, include_pole=True)
    elem, corners = sg.MeshLocator(mesh).locate_many(T.xyz())
    assert (elem >= 0).all()
    assert np.array_equal(corners, z["nodes"].astype(np.int64))


def _random_degenerate_grids(n, seed=777):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        nrows = int(rng.integers(4, 9))
        lats = np.sort(rng.uniform(-80, 80, nrows))[::-1]
        nl = [int(rng.choice([2, 3, 4, 5, 6, 8, 10, 12])) for _ in range(nrows)]
        nl[int(rng.integers(0, nrows))] = 2  # at least one 2-point row: elements in the plane y = 0
        out.append(tuple((float(round(a, 3)), b) for a, b in zip(lats, nl)))
    return out


@pytest.mark.parametrize("rows", _random_degenerate_grids(10))
def test_random_degenerate_meshes_match_the_oracle(gpu, rows):
    """Seeded random custom grids with 2-point rows: the device's per-target outcome (element /
    NotLocated / DegenerateTriangle) equals the oracle's restatement of MeshLocator.locate
    (oracle/locate_oracle.c: brute-force k = 8 / 32 nearest nodes, candidates in the reference's
    order, interp.py:90-117) except where the k-th nearest distance is tied (cKDTree order)."""
    sg = gpu
    from oracle import oracle as O

    S = sg.build_grid(sg.GridSpec(kind=sg.GridKind.CUSTOM, rows=rows))
    mesh = sg.generate_mesh(S, sg.blocks_partition(S, 1), 0, halo=0, include_pole=True)
    conn = mesh.element_connectivity
    for tname in ("O8", "F8"):
        xyz = sg.grid_from_name(tname).xyz()
        elem, _ = sg.MeshLocator(mesh).locate_many(xyz)
        oelem, _ = O.locate(mesh.node_xyz, conn.offsets, conn.indices, xyz)
        code = np.where(elem >= 0, 0, np.where(elem == -2, 2, 1))
        ocode = np.where(oelem >= 0, 0, np.where(oelem == -2, 2, 1))
        diff = np.flatnonzero((code != ocode) | ((code == 0) & (elem != oelem)))
        untied = [int(t) for t in diff if not _tied_at_k(mesh.node_xyz, xyz[t])]
        assert not untied, (tname, untied[:10], code[untied[:10]], ocode[untied[:10]])
        assert (ocode == 2).any()
