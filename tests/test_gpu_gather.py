"""gather_field / scatter_field on the device (functionspace.py:185-224)
against the unmodified reference's outputs (tests/golden/gather_scatter.npz, make_golden.py
`gather_scatter`): the gathered global array bitwise, every rank's scattered rows bitwise, and
the message counters (messages_sent, bytes_sent, messages_received) equal to the reference's
for P = 1, 2, 4 — with host-resident fields (one staging upload) and device-dirty fields (read
straight from HBM)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,levels", [("REAL64", 4), ("INT32", 3)])
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("device_dirty", [False, True])
def test_gather_scatter_equal_reference(gpu, golden, kind, levels, P, device_dirty):
    sg = gpu
    import paper_1908_07038_b200.functionspace as FS

    z = golden("gather_scatter")
    tag = kind.lower()
    gvals = z[f"{tag}_values"]
    g = sg.grid_from_name("O32")
    K = getattr(sg.Kind, kind)
    calls = {"rows_copy": 0}
    orig = FS._rows_copy

    def counting(*a, **k):
        calls["rows_copy"] += 1
        return orig(*a, **k)

    def program(ctx):
        c = ctx if ctx.nranks > 1 else None
        dist = sg.blocks_partition(g, ctx.nranks)
        mesh = sg.generate_mesh(g, dist, ctx.rank, halo=1, include_pole=True)
        fs = sg.NodeColumns(mesh, c)
        f = fs.create_field("n", levels, K)
        own = fs.owned_row_index()
        f.host[own] = gvals[mesh.node_global[own]]
        if device_dirty:
            f.allocate_device()
            with f.device_view(sg.Intent.READ_WRITE):
                pass
            f.host[:] = 0  # stale host: the gather must read HBM
        m0 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
        gathered = sg.gather_field(fs, f, c)
        m1 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
        sfs = sg.StructuredColumns(g, dist, ctx.rank)
        sf = sfs.create_field("s", levels, K)
        sg.scatter_field(sfs, sf, c, gvals[: g.npts] if ctx.rank == 0 else None)
        m2 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
        return gathered, np.array([np.subtract(m1, m0), np.subtract(m2, m1)]), sf.host.copy(), sf.state

    FS._rows_copy = counting
    try:
        res = sg.run_ranks(P, program, devices=[0])
    finally:
        FS._rows_copy = orig
    assert calls["rows_copy"] >= 1  # the device path ran
    assert np.array_equal(res[0][0].view(np.uint8), z[f"{tag}_p{P}_gathered"].view(np.uint8))
    assert all(r[0] is None for r in res[1:])
    for r in range(P):
        assert np.array_equal(res[r][1], z[f"{tag}_p{P}_r{r}_counters"]), r
        assert np.array_equal(res[r][2].view(np.uint8), z[f"{tag}_p{P}_r{r}_scattered"].view(np.uint8)), r
        assert res[r][3] is sg.MemoryState.HOST_ONLY


def test_scatter_dtype_quirk_stays_on_host(gpu):
    """A global array whose dtype differs from the field's keeps the reference behaviour
    (functionspace.py:207-224 casts on rank 0 and reinterprets bytes elsewhere): host path."""
    sg = gpu
    g = sg.grid_from_name("O8")
    vals = np.arange(g.npts * 2, dtype=np.int64).reshape(g.npts, 2)
    fs = sg.StructuredColumns(g, sg.blocks_partition(g, 1), 0)
    f = fs.create_field("x", 2)  # real64
    sg.scatter_field(fs, f, None, vals)
    assert np.array_equal(f.host, vals.astype(np.float64))


def _random_gs_cases(n, seed=4242):
    rng = np.random.default_rng(seed)
    grids = ["O8", "O16", "O24", "F8", "F12"]
    kinds = ["REAL64", "REAL32", "INT32", "INT64"]
    return [(str(rng.choice(grids)), int(rng.integers(1, 7)), str(rng.choice(kinds)), int(rng.choice([1, 2, 5, 137])),
             int(rng.integers(0, 3)), bool(rng.integers(0, 2))) for _ in range(n)]


@pytest.mark.parametrize("grid,P,kind,levels,halo,dirty", _random_gs_cases(16))
def test_random_gather_scatter_vs_reference_algorithm(gpu, grid, P, kind, levels, halo, dirty):
    """Seeded sweep: the device gather / scatter against the reference algorithm restated on
    the host (functionspace.py:185-224 — `_gather_host` / `_scatter_host`), bitwise, with the
    same message counters, on NodeColumns (any halo, host- or device-dirty fields) and
    StructuredColumns, every field kind."""
    sg = gpu
    import paper_1908_07038_b200.functionspace as FS
    from paper_1908_07038_b200.partition import PARTITIONERS

    g = sg.grid_from_name(grid)
    K = getattr(sg.Kind, kind)
    rng = np.random.default_rng(P * 10 + levels)
    gvals = (rng.normal(size=(g.npts + 2, levels)) * 1e6).astype(K.dtype)

    def program(ctx):
        c = ctx if ctx.nranks > 1 else None
        dist = PARTITIONERS["blocks" if halo != 1 else "equal_regions"](g, ctx.nranks)
        mesh = sg.generate_mesh(g, dist, ctx.rank, halo=halo, include_pole=True)
        fs = sg.NodeColumns(mesh, c)
        out = {}
        for name, fn in (("device", sg.gather_field), ("host", FS._gather_host)):
            f = fs.create_field("n", levels, K)
            own = fs.owned_row_index()
            f.host[own] = gvals[mesh.node_global[own]]
            if dirty:
                f.allocate_device()
                with f.device_view(sg.Intent.READ_WRITE):
                    pass
            m0 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
            got = fn(fs, f, c)
            out[name] = (got, np.subtract((ctx.messages_sent, ctx.bytes_sent, ctx.messages_received), m0))
        sfs = sg.StructuredColumns(g, dist, ctx.rank)
        for name, fn in (("sdevice", sg.scatter_field), ("shost", FS._scatter_host)):
            sf = sfs.create_field("s", levels, K)
            m0 = (ctx.messages_sent, ctx.bytes_sent, ctx.messages_received)
            fn(sfs, sf, c, gvals[: g.npts] if ctx.rank == 0 else None)
            out[name] = (sf.host.copy(), np.subtract((ctx.messages_sent, ctx.bytes_sent, ctx.messages_received), m0))
        return out

    res = sg.run_ranks(P, program, devices=[0])
    for r, o in enumerate(res):
        if r == 0:
            assert np.array_equal(o["device"][0].view(np.uint8), o["host"][0].view(np.uint8))
        else:
            assert o["device"][0] is None and o["host"][0] is None
        assert np.array_equal(o["device"][1], o["host"][1]), (r, o["device"][1], o["host"][1])
        assert np.array_equal(o["sdevice"][0].view(np.uint8), o["shost"][0].view(np.uint8))
        assert np.array_equal(o["sdevice"][1], o["shost"][1])
