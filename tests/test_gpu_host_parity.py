"""Host-side bit-exactness re-proved on the GPU box's host (run with ``-m gpu``).

The product builds its grids, latitudes, meshes and partitions on the host CPU (numpy's
arcsin/cos/sin and the native C++ setup code), and every GPU stencil rests on them.  The
CPU suite pins them against the reference's golden fixtures in the build container; numpy's
transcendental bits are host-dependent, so the same pins run here again,
marked ``gpu`` so the driver's GPU-box run executes them on that host:

* every oracle pin (tests/test_oracle.py) and every host-setup pin (tests/test_host_setup.py);
* the O1280 / O640 grids (latitudes, lonlats, xyz), the serial O1280 halo-2 mesh (cfg3's
  source) and O1280 P=8 halo-2 rank meshes, built by the product's own ``grid_from_name`` /
  ``generate_mesh``, against sha256 digests of the reference's arrays
  (tests/golden/mesh_digests.json, ``make_golden.py digests``);
* the O1280 -> O640 sample stencils located on the product's own grids (no injected
  latitudes).
"""
import functools
import hashlib
import json
import os

import numpy as np
import pytest

import test_host_setup as _host
import test_oracle as _oracle
from conftest import GOLDEN

W_TOL = 1e-13


def _on_gpu_host(fn):
    @functools.wraps(fn)
    def wrapper(*a, **k):
        return fn(*a, **k)

    return pytest.mark.gpu(wrapper)


for _mod, _prefix in ((_oracle, "oracle"), (_host, "host")):
    for _name in dir(_mod):
        if _name.startswith("test_"):
            globals()[f"test_{_prefix}_pin_{_name[5:]}_on_gpu_host"] = _on_gpu_host(getattr(_mod, _name))


def _digest(a) -> str:
    a = np.ascontiguousarray(a)
    return f"{a.dtype.str}:{'x'.join(map(str, a.shape))}:" + hashlib.sha256(a.tobytes()).hexdigest()


def _digests():
    path = os.path.join(GOLDEN, "mesh_digests.json")
    if not os.path.exists(path):
        pytest.skip("mesh_digests.json not generated")
    with open(path) as fh:
        return json.load(fh)


def _mesh_fields(mesh):
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


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["O1280", "O640"])
def test_own_grid_coordinates_bitwise(gpu, name):
    sg = gpu
    d = _digests()[f"grid_{name}"]
    G = sg.grid_from_name(name)
    assert G.npts == d["npts"]
    assert _digest(G.latitudes) == d["latitudes"]
    assert _digest(G.lonlats()) == d["lonlats"]
    assert _digest(G.xyz()) == d["xyz"]


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["mesh_O1280_p1_h2", "mesh_O1280_p8_h2_r0", "mesh_O1280_p8_h2_r3",
                                 "mesh_O1280_p8_h2_r7"])
def test_own_o1280_meshes_bitwise(gpu, key):
    sg = gpu
    dig = _digests()
    if key not in dig:
        pytest.skip(f"{key} digest not generated")
    _, _, parts, _, rank = (key.split("_") + [""])[:5]
    P = int(parts[1:])
    r = int(rank[1:]) if rank else 0
    S = sg.grid_from_name("O1280")
    mesh = sg.generate_mesh(S, sg.blocks_partition(S, P), r, halo=2, include_pole=True)
    got = _mesh_fields(mesh)
    want = dig[key]
    assert {k: got[k] == want[k] for k in want} == {k: True for k in want}


@pytest.mark.gpu
def test_o1280_o640_sample_on_own_grids(gpu, golden):
    """cfg3 sample stencils (lon 0/90/180/270 targets + 5000 random, the reference's
    MeshLocator) with the product's own latitudes, coordinates and mesh."""
    sg = gpu
    z = golden("o1280_o640_sample")
    S, T = sg.grid_from_name("O1280"), sg.grid_from_name("O640")
    assert np.array_equal(S.latitudes.view(np.uint64), z["src_lat"].view(np.uint64))
    assert np.array_equal(T.latitudes.view(np.uint64), z["tgt_lat"].view(np.uint64))
    dist = sg.blocks_partition(S, 1)
    mesh = sg.generate_mesh(S, dist, 0, halo=2, include_pole=True)
    w = sg.build_remap(sg.NodeColumns(mesh, None), T, sg.matching_partition(T, S, dist))
    ids = z["ids"]
    assert np.array_equal(w.target_global, np.arange(T.npts))
    assert np.array_equal(w.nodes[ids], z["corners"].astype(np.int64))
    assert np.array_equal(w.weights[ids].view(np.uint64), z["weights"].view(np.uint64))
