"""Device checksum / gather / scatter against the reference's golden digests
(tests/golden/checksum.npz: partition-invariant splitmix64 digests, functionspace.py:233-254)."""
import numpy as np
import pytest

import paper_1908_07038_b200 as sg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kind,levels", [("O32", "REAL64", 3), ("F8", "INT64", 2), ("O16", "REAL32", 5)])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_checksum_matches_reference(gpu, golden, name, kind, levels, P):
    z = golden("checksum")
    vals = z[f"{name}_values"]
    expect = z[f"{name}_p{P}"]
    g = sg.grid_from_name(name)
    k = getattr(sg.Kind, kind)

    def program(ctx):
        c = ctx if ctx.nranks > 1 else None
        dist = sg.blocks_partition(g, ctx.nranks)
        fs = sg.StructuredColumns(g, dist, ctx.rank)
        f = fs.create_field("x", levels, k)
        sg.scatter_field(fs, f, c, vals if ctx.rank == 0 else None)
        d1 = sg.checksum(fs, f, c)
        f.allocate_device()  # digest from the device mirror
        d1b = sg.checksum(fs, f, c)
        mesh = sg.generate_mesh(g, dist, ctx.rank, halo=1, include_pole=False)
        nfs = sg.NodeColumns(mesh, c)
        nf = nfs.create_field("y", levels, k)
        own = nfs.owned_row_index()
        nf.host[own] = vals[mesh.node_global[own]]
        d2 = sg.checksum(nfs, nf, c)
        gathered = sg.gather_field(fs, f, c)
        return d1, d1b, d2, gathered

    res = sg.run_ranks(P, program)
    assert res[0][0] == int(expect[0]) == res[0][1]
    assert res[0][2] == int(expect[1])
    assert np.array_equal(res[0][3], vals)
    assert sg.format_checksum(res[0][0]) == f"{int(expect[0]):016x}"


def test_scatter_gather_round_trip_and_nodecolumns(gpu):
    """test_functionspace.py:115-153: scatter -> gather is bitwise; gathering NodeColumns
    owned values over 2 ranks equals the serial gather."""
    sg = gpu
    g = sg.grid_from_name("O8")
    ref = np.random.default_rng(7).normal(size=(g.npts, 3))

    def worker(ctx):
        fs = sg.StructuredColumns(g, sg.blocks_partition(g, 4), ctx.rank)
        f = fs.create_field("v", levels=3)
        sg.scatter_field(fs, f, ctx, ref if ctx.rank == 0 else None)
        f.allocate_device()
        with f.device_view(sg.Intent.READ_WRITE):
            pass  # device-dirty: gather must read HBM
        return sg.gather_field(fs, f, ctx)

    assert np.array_equal(sg.run_ranks(4, worker)[0], ref)
    g8 = sg.grid_from_name("F8")
    serial = sg.generate_mesh(g8, sg.blocks_partition(g8, 1), 0)
    fs0 = sg.NodeColumns(serial, None)
    f0 = fs0.create_field("v")
    f0.host[:, 0] = np.sin(serial.node_global.astype(np.float64))
    expect = sg.gather_field(fs0, f0, None)

    def worker2(ctx):
        mesh = sg.generate_mesh(g8, sg.blocks_partition(g8, 2), ctx.rank, halo=1)
        fs = sg.NodeColumns(mesh, ctx)
        f = fs.create_field("v")
        f.host[:, 0] = np.sin(mesh.node_global.astype(np.float64))
        return sg.gather_field(fs, f, ctx)

    assert np.array_equal(sg.run_ranks(2, worker2)[0], expect)


def test_checksum_sensitivity(gpu):
    """test_functionspace.py:188-205: value, level and position sensitivity; format."""
    sg = gpu
    g = sg.grid_from_name("F4")
    fs = sg.StructuredColumns(g, sg.blocks_partition(g, 1), 0)
    f = fs.create_field("v", levels=2)
    f.host[:] = 1.0
    base = sg.checksum(fs, f, None)
    f.host[3, 0], f.host[3, 1] = 2.0, 1.0
    a = sg.checksum(fs, f, None)
    f.host[3, 0], f.host[3, 1] = 1.0, 2.0
    b = sg.checksum(fs, f, None)
    assert len({base, a, b}) == 3
    f.host[3, 1] += 1e-12
    assert sg.checksum(fs, f, None) != b
    assert sg.format_checksum(255) == "00000000000000ff" and len(sg.format_checksum(2**64 - 1)) == 16
