"""The fused distributed step with device-side signalling (csrc/step.cu, execute.FusedStep):
halo exchange over peer memory + apply as one kernel per rank, fenced by flag words that the
ranks write into each other's HBM instead of host or NCCL barriers.

One GPU cannot host ranks whose separate launches wait on each other (B200_PROFILING.md), so
P ranks are emulated as ONE launch over every rank's data (``launch_fused_steps``): the
protocol (epochs, ready/done words, the last-block count) and the peer reads run exactly as
with one GPU per rank, minus the tail wait — which the cooperative variant
(``launch_fused_steps_cooperative``, every block co-resident) runs too, on small problems.  Reference behaviour: halo_exchange
(functionspace.py:107-118) then apply_remap (interp.py:206-228), in the order of
cli.py:138-144; results must be bitwise equal to the oracle apply on the exchanged field."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ranks(sg, S, T, P, L, part, gvals, halo=2):
    from paper_1908_07038_b200.device import DeviceArray
    from paper_1908_07038_b200.partition import PARTITIONERS

    dist = PARTITIONERS[part](S, P)
    td = sg.matching_partition(T, S, dist)

    def prog(ctx):
        mesh = sg.generate_mesh(S, dist, ctx.rank, halo=halo, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        w = sg.build_remap(fs, T, td, ctx)
        src = DeviceArray(mesh.nb_nodes, L, np.float64)
        init = np.zeros((mesh.nb_nodes, L))
        own = fs.owned_row_index()
        init[own] = gvals[mesh.node_global[own]]
        src.upload(init)
        dst = DeviceArray(len(w), L, np.float64)
        return w, fs.exchange_plan, src, dst, mesh.nb_owned_nodes, mesh

    return sg.run_ranks(P, prog, devices=[0])


@pytest.mark.parametrize("S,T,P,L,part", [("O64", "O32", 2, 20, "blocks"), ("O64", "O32", 4, 137, "equal_regions"),
                                          ("O96", "O48", 8, 137, "equal_regions"), ("O64", "O32", 8, 3, "blocks"),
                                          ("F32", "F16", 3, 33, "blocks"), ("O32", "O64", 4, 137, "blocks"),
                                          ("O48", "O96", 8, 40, "equal_regions"), ("F16", "O32", 5, 200, "blocks"),
                                          ("O48", "O4", 8, 5, "blocks")])  # ranks without targets
def test_emulated_fused_step_bitwise(gpu, S, T, P, L, part):
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.device import synchronize
    from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps

    Sg, Tg = sg.grid_from_name(S), sg.grid_from_name(T)
    gvals = np.random.default_rng(11).normal(size=(Sg.npts + 2, L))
    ranks = _ranks(sg, Sg, Tg, P, L, part, gvals)
    steps = emulated_fused_steps([r[:4] for r in ranks])
    nsteps = 3
    for _ in range(nsteps):
        launch_fused_steps(steps)
    synchronize(0)
    if Sg.npts < Tg.npts:  # up-sampling: targets next to the partition boundary read peers' rows
        assert sum(s.n_boundary for s in steps) > 0
    for r, ((w, plan, src, dst, n_owned, mesh), st) in enumerate(zip(ranks, steps)):
        exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
        assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64)), f"rank {r}"
        assert not src.to_numpy()[n_owned:].any()  # ghosts never written: read from the owners
        assert st.check() == nsteps
        words = st.signal.read()
        assert words["error"] == 0 and words["count"] == 0 and words["current"] == nsteps
        for p in plan.recv:  # every owner published epoch nsteps to me
            assert words["ready"][p] == nsteps
        for p in plan.send:  # every reader of my rows finished epoch nsteps
            assert words["done"][p] == nsteps


def test_single_rank_step_equals_apply(gpu):
    """P = 1 (no peers): the real-mode launch (n = 1, wait_done = 1) is the plain apply."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.execute import FusedStep, Signal

    Sg, Tg = sg.grid_from_name("O48"), sg.grid_from_name("O24")
    L = 137
    gvals = np.random.default_rng(5).normal(size=(Sg.npts + 2, L))
    (w, plan, src, dst, n_owned, mesh), = _ranks(sg, Sg, Tg, 1, L, "blocks", gvals)
    sig = Signal(0, 1, 0)
    st = FusedStep(w, plan, src, dst, sig, [(src.ptr, src.pitch, 0)], [(sig.ptr, b"")])
    for _ in range(2):
        st.launch()
    assert st.check() == 2 and st.n_boundary == 0 and st.m == len(w)
    exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
    assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64))


def test_missing_peer_times_out_instead_of_hanging(gpu):
    """A rank whose owner never publishes its rows does not hang: the bounded wait (1 ms here)
    sets the error word and sg_step_check raises."""
    sg = gpu
    from paper_1908_07038_b200.device import synchronize
    from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps

    Sg, Tg = sg.grid_from_name("O32"), sg.grid_from_name("O16")
    gvals = np.zeros((Sg.npts + 2, 4))
    Tg = sg.grid_from_name("O48")  # finer targets: rank 0 has boundary targets
    ranks = _ranks(sg, Sg, Tg, 2, 4, "blocks", gvals)
    steps = emulated_fused_steps([r[:4] for r in ranks])
    assert steps[0].n_boundary > 0
    steps[0].set_timeout(1e-3)
    launch_fused_steps(steps[:1])  # rank 1 never runs
    synchronize(0)
    with pytest.raises(sg.SpheregridError, match="timed out"):
        steps[0].check()


def test_step_refuses_bad_launches(gpu):
    sg = gpu
    from paper_1908_07038_b200 import _native as N
    from paper_1908_07038_b200.execute import emulated_fused_steps

    Sg, Tg = sg.grid_from_name("O32"), sg.grid_from_name("O16")
    ranks = _ranks(sg, Sg, Tg, 2, 4, "blocks", np.zeros((Sg.npts + 2, 4)))
    steps = emulated_fused_steps([r[:4] for r in ranks])
    arr = np.array([s.handle for s in steps], np.uint64)
    with pytest.raises(N.NativeError, match="wait_done"):  # ranks of one launch cannot wait for each other
        N.call("sg_step_launch", N.ptr(arr), 2, 1, 0)


@pytest.mark.parametrize("grid,P,halo,part,kind,levels", [("O32", 2, 1, "blocks", "REAL64", 137),
                                                         ("O48", 4, 2, "equal_regions", "INT32", 3),
                                                         ("F16", 8, 3, "equal_regions", "REAL32", 33),
                                                         ("O24", 3, 2, "blocks", "INT64", 1),
                                                         ("O32", 5, 2, "blocks", "REAL64", 300)])
def test_emulated_signalled_exchange(gpu, grid, P, halo, part, kind, levels):
    """The halo exchange alone as one signalled pull kernel per rank (sg_exchange_*), P ranks in
    one launch on one GPU: every ghost row equals its owner's values (functionspace.py:107-118),
    owned rows untouched, signal words = epochs, for every field kind and level count."""
    sg = gpu
    from paper_1908_07038_b200.device import DeviceArray, synchronize
    from paper_1908_07038_b200.execute import emulated_exchanges, launch_exchanges
    from paper_1908_07038_b200.partition import PARTITIONERS

    S = sg.grid_from_name(grid)
    dist = PARTITIONERS[part](S, P)
    K = getattr(sg.Kind, kind)

    def prog(ctx):
        mesh = sg.generate_mesh(S, dist, ctx.rank, halo=halo, include_pole=True)
        plan = sg.NodeColumns(mesh, ctx).exchange_plan
        expect = (mesh.node_global[:, None] * 7 + np.arange(levels)[None, :] % 5).astype(K.dtype)
        d = DeviceArray(mesh.nb_nodes, levels, K.dtype)
        d.upload(np.where(mesh.node_ghost[:, None], 0, expect).astype(K.dtype))
        return plan, d, expect

    ranks = sg.run_ranks(P, prog, devices=[0])
    xs = emulated_exchanges([(plan, d) for plan, d, _ in ranks])
    for _ in range(2):
        launch_exchanges(xs)
    synchronize(0)
    for (plan, d, expect), x in zip(ranks, xs):
        assert np.array_equal(d.to_numpy(), expect)
        w = x.signal.read()
        assert w["epoch"] == 2 and w["error"] == 0 and w["count"] == 0
        assert all(w["ready"][p] == 2 for p in plan.recv) and all(w["done"][p] == 2 for p in plan.send)


def test_signalled_exchange_times_out_without_owner(gpu):
    sg = gpu
    from paper_1908_07038_b200.device import DeviceArray, synchronize
    from paper_1908_07038_b200.execute import emulated_exchanges, launch_exchanges

    S = sg.grid_from_name("O16")
    dist = sg.blocks_partition(S, 2)

    def prog(ctx):
        mesh = sg.generate_mesh(S, dist, ctx.rank, halo=1, include_pole=True)
        return sg.NodeColumns(mesh, ctx).exchange_plan, DeviceArray(mesh.nb_nodes, 2, np.float64)

    xs = emulated_exchanges(sg.run_ranks(2, prog, devices=[0]))
    xs[0].set_timeout(1e-3)
    launch_exchanges(xs[:1])  # rank 1 never publishes its rows
    synchronize(0)
    with pytest.raises(sg.SpheregridError, match="timed out"):
        xs[0].check()


def _random_step_cases(n, seed=9117):
    rng = np.random.default_rng(seed)
    grids = ["O16", "O24", "O32", "O48", "F8", "F16", "F24"]
    out = []
    for _ in range(n):
        s, t = rng.choice(grids, 2, replace=False)
        out.append((str(s), str(t), int(rng.integers(2, 9)), int(rng.integers(1, 4)),
                    str(rng.choice(["blocks", "equal_regions"])), int(rng.choice([1, 7, 64, 137, 161]))))
    return out


@pytest.mark.parametrize("S,T,P,halo,part,L", _random_step_cases(14))
def test_random_fused_steps_and_exchanges(gpu, S, T, P, halo, part, L):
    """Seeded random sweep (grid pairs up and down, 2-8 ranks, halo 1-3, both decompositions,
    1-161 levels): per rank the fused step equals the oracle apply on the exchanged field and
    the signalled exchange leaves every ghost equal to its owner, three epochs in a row.
    Thin halos can leave targets without a containing element: those runs use the reference's
    nearest-node fallback rows (allow_fallback), which the step applies like any stencil."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, synchronize
    from paper_1908_07038_b200.execute import (emulated_exchanges, emulated_fused_steps, launch_exchanges,
                                               launch_fused_steps)
    from paper_1908_07038_b200.partition import PARTITIONERS

    Sg, Tg = sg.grid_from_name(S), sg.grid_from_name(T)
    dist = PARTITIONERS[part](Sg, P)
    td = sg.matching_partition(Tg, Sg, dist)
    gvals = np.random.default_rng(P * 100 + halo).normal(size=(Sg.npts + 2, L))

    def prog(ctx):
        mesh = sg.generate_mesh(Sg, dist, ctx.rank, halo=halo, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        w = sg.build_remap(fs, Tg, td, ctx, allow_fallback=True)
        init = np.where(mesh.node_ghost[:, None], 0.0, gvals[mesh.node_global])
        a, b = DeviceArray(mesh.nb_nodes, L, np.float64), DeviceArray(mesh.nb_nodes, L, np.float64)
        a.upload(init)
        b.upload(init)
        return mesh, fs.exchange_plan, w, a, b, DeviceArray(len(w), L, np.float64)

    ranks = sg.run_ranks(P, prog, devices=[0])
    xs = emulated_exchanges([(r[1], r[3]) for r in ranks])
    steps = emulated_fused_steps([(r[2], r[1], r[4], r[5]) for r in ranks])
    for _ in range(3):
        launch_exchanges(xs)
        launch_fused_steps(steps)
    synchronize(0)
    for mesh, plan, w, a, b, out in ranks:
        assert np.array_equal(a.to_numpy(), gvals[mesh.node_global])
        exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
        assert np.array_equal(out.to_numpy().view(np.uint64), exp.view(np.uint64))
    assert all(x.check() == 3 for x in xs) and all(st.check() == 3 for st in steps)


def test_signalled_launches_replay_from_a_cuda_graph(gpu):
    """The N>1 step is captured once into a CUDA graph and replayed (bench.py run_multi): the
    signal kernels and the programmatically dependent step / pull kernels (PDL) captured on a
    stream replay bitwise, with the epochs advancing once per replay."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, Graph, Stream
    from paper_1908_07038_b200.execute import (emulated_exchanges, emulated_fused_steps, launch_exchanges,
                                               launch_fused_steps)

    Sg, Tg = sg.grid_from_name("O32"), sg.grid_from_name("O64")
    L = 9
    gvals = np.random.default_rng(3).normal(size=(Sg.npts + 2, L))
    ranks = _ranks(sg, Sg, Tg, 3, L, "equal_regions", gvals)
    xfields = [DeviceArray(r[2].shape[0], L, np.float64) for r in ranks]
    for xf, r in zip(xfields, ranks):
        xf.upload(np.where(r[5].node_ghost[:, None], 0.0, gvals[r[5].node_global]))
    xs = emulated_exchanges([(r[1], xf) for r, xf in zip(ranks, xfields)])
    steps = emulated_fused_steps([r[:4] for r in ranks])
    st = Stream(0)

    def body():
        launch_exchanges(xs, st.stream)
        launch_fused_steps(steps, st.stream)

    g = Graph(0, st.stream, body)
    for _ in range(4):
        g.launch(st.stream)
    st.synchronize()
    for (w, plan, src, dst, n_owned, mesh), xf in zip(ranks, xfields):
        assert np.array_equal(xf.to_numpy(), gvals[mesh.node_global])
        exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
        assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64))
    assert all(x.check() == 4 for x in xs) and all(s.check() == 4 for s in steps)


def test_many_epochs_share_one_signal(gpu):
    """200 rounds of exchange + step per rank sharing ONE signal per rank (epochs advance by two
    per round): counters reset every epoch, no drift, results stay bitwise."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, synchronize
    from paper_1908_07038_b200.execute import (FusedStep, Signal, SignalledExchange, launch_exchanges,
                                               launch_fused_steps)

    Sg, Tg = sg.grid_from_name("O24"), sg.grid_from_name("O48")
    L, P = 5, 4
    gvals = np.random.default_rng(1).normal(size=(Sg.npts + 2, L))
    ranks = _ranks(sg, Sg, Tg, P, L, "equal_regions", gvals)
    sigs = [Signal(0, P, r) for r in range(P)]
    uuid = sg._native.device_uuid(0)
    psig = [(s.ptr, uuid) for s in sigs]
    xf = []
    for r in ranks:
        d = DeviceArray(r[2].shape[0], L, np.float64)
        d.upload(np.where(r[5].node_ghost[:, None], 0.0, gvals[r[5].node_global]))
        xf.append(d)
    xinfo = [(d.ptr, d.pitch, 0) for d in xf]
    sinfo = [(r[2].ptr, r[2].pitch, 0) for r in ranks]
    xs = [SignalledExchange(r[1], xf[i], sigs[i], xinfo, psig) for i, r in enumerate(ranks)]
    steps = [FusedStep(r[0], r[1], r[2], r[3], sigs[i], sinfo, psig) for i, r in enumerate(ranks)]
    for _ in range(200):
        launch_exchanges(xs)
        launch_fused_steps(steps)
    synchronize(0)
    for i, (w, plan, src, dst, n_owned, mesh) in enumerate(ranks):
        assert np.array_equal(xf[i].to_numpy(), gvals[mesh.node_global])
        exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
        assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64))
        words = sigs[i].read()
        assert words["epoch"] == 400 and words["count"] == 0 and words["error"] == 0


@pytest.mark.parametrize("P,part", [(4, "blocks"), (6, "equal_regions")])
def test_emulated_fused_step_structured_bilinear(gpu, P, part):
    """The fused step with 4-point structured-bilinear stencils (cfg5's method, csrc/bilinear.cu):
    bitwise equal to the oracle's 4-point apply ((w0 a + w1 b) + w2 c) + w3 d on the exchanged
    field, P ranks emulated as one launch."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, synchronize
    from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps
    from paper_1908_07038_b200.partition import PARTITIONERS

    S, T = sg.grid_from_name("O48"), sg.grid_from_name("O32")
    L = 21
    dist = PARTITIONERS[part](S, P)
    td = sg.matching_partition(T, S, dist)
    gvals = np.random.default_rng(12).normal(size=(S.npts + 2, L))

    def prog(ctx):
        mesh = sg.generate_mesh(S, dist, ctx.rank, halo=2, include_pole=True)
        fs = sg.NodeColumns(mesh, ctx)
        w = sg.build_bilinear(fs, T, td, ctx)
        src = DeviceArray(mesh.nb_nodes, L, np.float64)
        src.upload(np.where(mesh.node_ghost[:, None], 0.0, gvals[mesh.node_global]))
        return w, fs.exchange_plan, src, DeviceArray(len(w), L, np.float64), mesh

    ranks = sg.run_ranks(P, prog, devices=[0])
    steps = emulated_fused_steps([r[:4] for r in ranks])
    launch_fused_steps(steps)
    synchronize(0)
    assert all(w.nodes.shape[1] == 4 for w, *_ in ranks)
    for w, plan, src, dst, mesh in ranks:
        exp = O.apply_remap_k(w.nodes, w.weights, gvals[mesh.node_global])
        assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64))


@pytest.mark.parametrize("S,T,P,L,part", [("O16", "O32", 2, 7, "blocks"), ("O16", "O24", 4, 33, "equal_regions"),
                                          ("F8", "O24", 3, 137, "blocks")])  # grids of <= 32 x 148 blocks
def test_cooperative_emulation_runs_the_tail_waits(gpu, S, T, P, L, part):
    """The finisher's tail wait (wait_done = 1: an owner waits for every reader's done word
    before the next epoch may overwrite its rows) exercised on one GPU: every rank in ONE
    cooperative launch (all blocks co-resident), so a rank's last block may spin on the done
    words that other ranks' blocks of the same grid write.  Exchange + step, three epochs,
    bitwise vs the oracle, done words = epochs."""
    sg = gpu
    from oracle import oracle as O
    from paper_1908_07038_b200.device import DeviceArray, synchronize
    from paper_1908_07038_b200.execute import (emulated_exchanges, emulated_fused_steps,
                                               launch_exchanges_cooperative, launch_fused_steps_cooperative)

    Sg, Tg = sg.grid_from_name(S), sg.grid_from_name(T)
    gvals = np.random.default_rng(P * 31 + L).normal(size=(Sg.npts + 2, L))
    ranks = _ranks(sg, Sg, Tg, P, L, part, gvals)
    xf = []
    for r in ranks:
        d = DeviceArray(r[2].shape[0], L, np.float64)
        d.upload(np.where(r[5].node_ghost[:, None], 0.0, gvals[r[5].node_global]))
        xf.append(d)
    xs = emulated_exchanges([(r[1], d) for r, d in zip(ranks, xf)])
    steps = emulated_fused_steps([r[:4] for r in ranks])
    for _ in range(3):
        launch_exchanges_cooperative(xs)
        launch_fused_steps_cooperative(steps)
    synchronize(0)
    assert sum(s.n_boundary for s in steps) > 0
    for i, (w, plan, src, dst, n_owned, mesh) in enumerate(ranks):
        assert np.array_equal(xf[i].to_numpy(), gvals[mesh.node_global])
        exp = O.apply_remap(w.nodes, w.weights, gvals[mesh.node_global])
        assert np.array_equal(dst.to_numpy().view(np.uint64), exp.view(np.uint64)), f"rank {i}"
        for words in (xs[i].signal.read(), steps[i].signal.read()):
            assert words["epoch"] == 3 and words["error"] == 0 and words["count"] == 0
            assert all(words["done"][p] == 3 for p in plan.send)
            assert all(words["ready"][p] == 3 for p in plan.recv)


def test_tail_wait_times_out_when_a_reader_never_reads(gpu):
    """wait_done = 1 really waits: rank 0 alone (owners' ready words published ahead, so only
    the tail wait can block) waits for its readers' done words, which never come; the bounded
    wait sets the error word instead of hanging."""
    sg = gpu
    from paper_1908_07038_b200.device import synchronize
    from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps

    Sg, Tg = sg.grid_from_name("O32"), sg.grid_from_name("O48")
    ranks = _ranks(sg, Sg, Tg, 2, 4, "blocks", np.zeros((Sg.npts + 2, 4)))
    steps = emulated_fused_steps([r[:4] for r in ranks])
    assert ranks[0][1].send  # rank 1 reads rank 0's rows
    steps[0].signal.publish_owners_ahead(1)
    steps[0].set_timeout(1e-3)
    launch_fused_steps(steps[:1], wait_done=True)
    synchronize(0)
    with pytest.raises(sg.SpheregridError, match="timed out"):
        steps[0].check()


def test_cooperative_launch_refuses_a_grid_that_does_not_fit(gpu):
    sg = gpu
    from paper_1908_07038_b200 import _native as N
    from paper_1908_07038_b200.execute import emulated_fused_steps, launch_fused_steps_cooperative

    Sg, Tg = sg.grid_from_name("O400"), sg.grid_from_name("O800")
    ranks = _ranks(sg, Sg, Tg, 2, 1, "blocks", np.zeros((Sg.npts + 2, 1)))
    steps = emulated_fused_steps([r[:4] for r in ranks])
    with pytest.raises(N.NativeError, match="co-resident"):
        launch_fused_steps_cooperative(steps)
