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
