"""Executor host logic on CPU through the numpy libcq double (tests/fakecq.py):
single process with several nodes per device / several devices, and a real
2-rank torch.distributed gloo run in which NCCL groups travel over gloo.
Results must equal the reference's golden outputs bit for bit."""

import json
import os
import socket

import numpy as np
import pytest

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import _native as N
from paper_2505_06022_b200 import executor as E
from paper_2505_06022_b200 import workloads as W
from fakecq import FakeLib, GlooTransport, LocalTransport
from oracle import dsl
from progjson import graph_of, load_arrays, program_from_json

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "programs.json")) as fh:
    PROGRAMS = json.load(fh)
EXPECTED = load_arrays(os.path.join(GOLD, "expected.npz"))
OK_IDX = [i for i, e in enumerate(PROGRAMS) if e["error"] is None]


@pytest.fixture
def fake(monkeypatch):
    def install(ndev=1, transport=None):
        lib = FakeLib(ndev, transport or LocalTransport())
        monkeypatch.setattr(N, "_lib", lib)
        E._pinned.clear()
        return lib
    return install


def test_jit_codegen_compiles_every_golden_body(fake, monkeypatch):
    """Force the DSL->CUDA JIT for every launch: each golden program's
    generated kernel must compile with NVRTC for sm_100a (real compiler, no
    GPU needed) and the run must still match the reference bit for bit."""
    from paper_2505_06022_b200 import jit
    monkeypatch.setattr(jit, "MODE", "1")
    lib = fake(1)
    for idx in OK_IDX[::3]:
        entry = PROGRAMS[idx]
        buffers, tasks = program_from_json(entry["program"])
        res = E.run(cq.generate_commands(graph_of(buffers, tasks), entry["nodes"]))
        for name in buffers:
            assert dsl.same_bits(res.buffers[name], EXPECTED[f"p{idx}__{name}"]), (entry["name"], name)
    assert lib.jit_compiled > 0 and "jit" in lib.launches


@pytest.mark.parametrize("idx", OK_IDX)
def test_golden_programs_single_process(fake, idx):
    entry = PROGRAMS[idx]
    for ndev, nodes in ((1, entry["nodes"]), (2, 5)):
        fake(ndev)
        buffers, tasks = program_from_json(entry["program"])
        plan = cq.generate_commands(graph_of(buffers, tasks), nodes)
        res = E.run(plan, placement=E.Placement(1, 0, tuple(range(ndev))))
        for name in buffers:
            assert dsl.same_bits(res.buffers[name], EXPECTED[f"p{idx}__{name}"]), (entry["name"], name)


def test_error_programs_raise_reference_error(fake):
    fake(1)
    for entry in PROGRAMS:
        if entry["error"] is None:
            continue
        buffers, tasks = program_from_json(entry["program"])
        with pytest.raises(cq.ClusterqError) as info:
            E.run(cq.generate_commands(graph_of(buffers, tasks), entry["nodes"]))
        assert type(info.value).__name__ == entry["error"]


def test_wave_interior_boundary_split_and_session_rerun(fake):
    lib = fake(1)
    h, w = 48, 40
    u0 = np.random.default_rng(4).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=4, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), 3)
    s = E.Session(plan, E.Placement(1, 0, (0,)))
    s.execute(upload=True)
    s.synchronize()
    first = s.results()
    s.recycle()
    # nodes 1..2 get halo rows each step: chunks split into 3 launches
    launches = lib.launches.count("wave5")
    assert launches > 3 * 4
    # replay on resident data (benchmark mode): same launches, no uploads
    s.execute(upload=False)
    s.synchronize()
    assert lib.launches.count("wave5") == 2 * launches
    s.recycle()
    # a fresh upload reproduces the first result exactly
    s.execute(upload=True)
    s.synchronize()
    again = s.results()
    s.close()
    from oracle import native as onat
    u, up = onat.wave_run(u0, u0, 4, 0.25)
    assert dsl.same_bits(first["u"], u) and dsl.same_bits(first["up"], up)
    assert dsl.same_bits(again["u"], u) and dsl.same_bits(again["up"], up)


# ------------------------------------------------------- 2 ranks over gloo

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _nbody_prog():
    pos, vel = W.nbody_inputs(96)
    return W.nbody_program(96, steps=2, pos=pos, vel=vel)


def _sgemm_prog():
    a, b = W.sgemm_inputs(40, 24, 16)
    return W.sgemm_program(40, 24, 16, a=a, b=b)


def _rank_main(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = FakeLib(1, GlooTransport())
    N._lib = lib
    pl = E.Placement(world, rank, (0,))
    results = {}
    h, w = 37, 24
    u0 = np.random.default_rng(9).uniform(0, 1, (h, w)).astype(np.float32)
    for nodes in (2, 3):
        prog = W.wave_program(h, w, steps=5, kind="float32", u0=u0, up0=u0)
        res = E.run(cq.generate_commands(prog.graph(), nodes), placement=pl)
        if rank == 0:
            results[f"wave{nodes}_u"] = res.buffers["u"]
            results[f"wave{nodes}_up"] = res.buffers["up"]
        loc = E.run(cq.generate_commands(prog.graph(), nodes), placement=pl, gather="local")
        results[f"local{nodes}_r{rank}"] = loc.buffers.get("u", np.zeros(0))
    # temporally blocked chain: the KL-row halo exchange crosses ranks
    fu0 = np.random.default_rng(10).uniform(0, 1, (160, 32)).astype(np.float32)
    for nodes in (2, 3):
        prog = W.wave_program(160, 32, steps=14, kind="float32", u0=fu0, up0=fu0)
        sess = E.Session(cq.generate_commands(prog.graph(), nodes), pl)
        assert [b.kl for b in sess.chains[0].blocks] == [4, 8]
        sess.execute(upload=True)
        sess.synchronize()
        res = sess.results()
        sess.close()
        if rank == 0:
            results[f"fwave{nodes}_u"], results[f"fwave{nodes}_up"] = res["u"], res["up"]
    for idx in OK_IDX[::6]:
        entry = PROGRAMS[idx]
        buffers, tasks = program_from_json(entry["program"])
        res = E.run(cq.generate_commands(graph_of(buffers, tasks), entry["nodes"]), placement=pl)
        if rank == 0:
            for name in buffers:
                results[f"g{idx}__{name}"] = res.buffers[name]
    # N-body: the 'all' mapper's pushes = an all-gather group per step;
    # sgemm: A slabs scattered, B broadcast (host-init lowering at each rank)
    for nodes in (2, 3):
        before = len(lib.launches)
        res = E.run(cq.generate_commands(_nbody_prog().graph(), nodes), placement=pl)
        new = lib.launches[before:]
        # 2 nodes = 2 ranks: one in-place all-gather per later step, and the
        # kick split into held / arriving j columns
        results[f"nbody{nodes}_allgathers_r{rank}"] = np.array(
            [sum(1 for x in new if isinstance(x, tuple) and x[0] == "allgather"),
             sum(1 for x in new if x == "nbody.partial")])
        if rank == 0:
            results[f"nbody{nodes}_P"], results[f"nbody{nodes}_V"] = res.buffers["P"], res.buffers["V"]
        res = E.run(cq.generate_commands(_sgemm_prog().graph(), nodes), placement=pl)
        if rank == 0:
            results[f"sgemm{nodes}_C"] = res.buffers["C"]
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **results)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo(tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    r0 = dict(np.load(tmp_path / "rank0.npz"))
    r1 = dict(np.load(tmp_path / "rank1.npz"))
    from oracle import native as onat
    h, w = 37, 24
    u0 = np.random.default_rng(9).uniform(0, 1, (h, w)).astype(np.float32)
    u, up = onat.wave_run(u0, u0, 5, 0.25)
    for nodes in (2, 3):
        assert dsl.same_bits(r0[f"wave{nodes}_u"], u) and dsl.same_bits(r0[f"wave{nodes}_up"], up)
    fu0 = np.random.default_rng(10).uniform(0, 1, (160, 32)).astype(np.float32)
    fu, fup = onat.wave_run(fu0, fu0, 14, 0.25)
    for nodes in (2, 3):
        assert dsl.same_bits(r0[f"fwave{nodes}_u"], fu) and dsl.same_bits(r0[f"fwave{nodes}_up"], fup)
    # gather="local": each rank holds exactly its own final rows
    assert dsl.same_bits(r0["local2_r0"][:19], u[:19]) and dsl.same_bits(r1["local2_r1"][19:], u[19:])
    for key, val in r0.items():
        if key.startswith("g"):
            idx, name = key[1:].split("__")
            assert dsl.same_bits(val, EXPECTED[f"p{idx}__{name}"]), key
    # the distributed runs equal a single-process run of the same double
    N._lib = FakeLib(1, LocalTransport())
    single_nb = E.run(cq.generate_commands(_nbody_prog().graph(), 1), placement=E.Placement(1, 0, (0,)))
    single_mm = E.run(cq.generate_commands(_sgemm_prog().graph(), 1), placement=E.Placement(1, 0, (0,)))
    N._lib = None
    for r in (r0, r1):
        ag2, part2 = r[f"nbody2_allgathers_r{r is r1:d}"]
        ag3, _ = r[f"nbody3_allgathers_r{r is r1:d}"]
        assert ag2 == 1 and part2 >= 2 and ag3 == 0   # 3 nodes on 2 ranks: send/recv groups
    for nodes in (2, 3):
        assert dsl.same_bits(r0[f"nbody{nodes}_P"], single_nb.buffers["P"])
        assert dsl.same_bits(r0[f"nbody{nodes}_V"], single_nb.buffers["V"])
        assert dsl.same_bits(r0[f"sgemm{nodes}_C"], single_mm.buffers["C"])


def test_graph_capture_replays_same_commands(fake):
    lib = fake(1)
    h, w = 40, 32
    u0 = np.random.default_rng(4).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=4, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), 3)
    s = E.Session(plan, E.Placement(1, 0, (0,)))
    s.execute(upload=True)
    s.synchronize()
    base = lib.launches.count("wave5")
    s.capture()
    assert lib.launches.count("wave5") == base  # capture records, runs nothing
    s.replay(2)
    s.synchronize()
    assert lib.launches.count("wave5") == 3 * base
    assert s.graph_log == [] and s.graph_events == []
    # timed capture: the launch log survives, its events stay out of the pool
    s.capture(timed=True)
    assert len([x for x in s.graph_log if x[0] == "wave5"]) == base
    held = set(s.graph_events)
    assert held and not held & {ev for pool in s.free_events.values() for ev in pool}
    s.replay(1)
    s.synchronize()
    assert lib.launches.count("wave5") == 4 * base
    s.close()
    assert s.graph is None and s.graph_events == []


def test_failed_capture_restores_fused_views(fake):
    """A capture that fails part-way through a fused chain (here: the
    second block's launch) leaves no current / alternate swap behind: the
    stream replay that follows continues the simulation exactly."""
    from oracle import native as onat
    lib = fake(1)
    h, w, steps = 288, 64, 20          # 3 out-of-place blocks: KL4 + 2 x KL8
    u0 = np.random.default_rng(21).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=u0)
    s = E.Session(cq.generate_commands(prog.graph(), 3), E.Placement(1, 0, (0,)))
    assert [b.kl for b in s.chains[0].blocks] == [4, 8, 8]
    s.execute(upload=True)
    s.synchronize()
    s.recycle()
    real = lib.cq_wave5_fused_bounded
    calls = []

    def failing(*args):
        if lib.capturing is not None:
            calls.append(1)
            if len(calls) == 4:        # block 2's first launch (3 nodes per block)
                return N.CQ_ERR_ARG
        return real(*args)
    lib.cq_wave5_fused_bounded = failing
    with pytest.raises(cq.NativeError):
        s.capture()
    lib.cq_wave5_fused_bounded = real
    s.execute(upload=False)
    s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, u0, 2 * steps, 0.25)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


# ------------------------------------------- temporally blocked wave chains

@pytest.mark.parametrize("steps,nodes,ndev", [(22, 1, 1), (22, 3, 1), (16, 4, 2), (9, 2, 1), (100, 3, 2)])
def test_fused_wave_chain_matches_oracle(fake, monkeypatch, steps, nodes, ndev):
    """Fused blocks (a KL=4 block for a remaining quarter first, then KL=8
    blocks; odd block counts included) + plain leftovers give the per-step
    result bit for bit, with nodes sharing or spanning devices."""
    from paper_2505_06022_b200 import fusion
    from oracle import native as onat
    lib = fake(ndev)
    h, w = 200, 64
    u0 = np.random.default_rng(11).uniform(0, 1, (h, w)).astype(np.float32)
    up0 = np.random.default_rng(12).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=up0)
    plan = cq.generate_commands(prog.graph(), nodes)
    s = E.Session(plan, E.Placement(1, 0, tuple(range(ndev))))
    assert (len(s.chains) == 1) == (steps >= 8)
    if s.chains:
        ch = s.chains[0]
        kls = [b.kl for b in ch.blocks]
        assert kls.count(4) <= 1 and (kls.count(4) == 0 or kls[0] == 4)
        assert sum(b.kl for b in ch.blocks) + len(ch.plain) == steps
    s.execute(upload=True)
    s.synchronize()
    res = s.results()
    trace, _ = s.trace()
    s.close()
    u, up = onat.wave_run(u0, up0, steps, 0.25)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)
    if steps >= 8:
        assert "wave5_fused" in lib.launches
    # one trace event per execute and per push command, fused or not
    assert sum(1 for e in trace if e.kind == "execute") == steps * nodes
    n_push = sum(1 for c in plan.commands if type(c).__name__ == "PushCommand")
    assert sum(1 for e in trace if e.kind == "push") == n_push


def test_fused_chain_magnitude_bounds_wiring(fake):
    """Every fused launch of a float32 chain writes its node's bound slot for
    the block; only interior launches after the first block read the
    previous block's slot (edges read received rows: exact form)."""
    lib = fake(1)
    h, w = 200, 64
    u0 = np.random.default_rng(13).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=24, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), 2)
    s = E.Session(plan, E.Placement(1, 0, (0,)))
    ch = s.chains[0]
    s.execute(upload=True)
    s.synchronize()
    s.close()
    slots = {node: s._amax[(0, node)] for node in ch.rows}
    bounds = lib.fused_bounds
    # per block: node 0 (interior + bottom edge), node 1 (top edge + interior)
    per_block = len(bounds) // len(ch.blocks)
    assert per_block * len(ch.blocks) == len(bounds) == 4 * len(ch.blocks)
    for bi in range(len(ch.blocks)):
        launches = bounds[bi * per_block:(bi + 1) * per_block]
        outs = {o for _i, o in launches}
        assert outs == {slots[n] + 4 * (bi + 1) for n in slots}
        reads = [i for i, _o in launches if i]
        if bi == 0:
            assert reads == []
        else:
            assert sorted(reads) == sorted(slots[n] + 4 * bi for n in slots)


def test_fused_chain_disabled_and_graph_replay(fake, monkeypatch):
    from oracle import native as onat
    lib = fake(1)
    h, w, steps = 160, 32, 12
    u0 = np.random.default_rng(5).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), 2)
    monkeypatch.setenv("CQ_WAVE_FUSE", "0")
    s0 = E.Session(plan, E.Placement(1, 0, (0,)))
    assert s0.chains == []
    s0.close()
    monkeypatch.delenv("CQ_WAVE_FUSE")
    s = E.Session(plan, E.Placement(1, 0, (0,)))
    assert [b.kl for b in s.chains[0].blocks] == [4, 8]
    s.execute(upload=True)
    s.synchronize()
    s.recycle()
    views0 = {k: v.ptr for k, v in s.views.items()}
    s.capture()
    # an even number of out-of-place blocks: the captured replay starts and
    # ends on the same allocations
    assert {k: v.ptr for k, v in s.views.items()} == views0
    s.replay(2)
    s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, u0, 3 * steps, 0.25)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


def test_odd_fused_chain_graph_replays_alternate(fake):
    """An odd number of out-of-place blocks ends a run on the alternate
    allocations: capture records two graphs (one from each side), replay
    alternates them and the views follow, so any number of replays continues
    the simulation."""
    from oracle import native as onat
    fake(1)
    h, w, steps = 160, 32, 20
    u0 = np.random.default_rng(6).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=u0)
    s = E.Session(cq.generate_commands(prog.graph(), 2), E.Placement(1, 0, (0,)))
    assert [b.kl for b in s.chains[0].blocks] == [4, 8, 8]
    s.execute(upload=True)
    s.synchronize()
    s.recycle()
    views0 = {k: v.ptr for k, v in s.views.items()}
    s.capture()
    assert len(s.graphs) == 2
    assert {k: v.ptr for k, v in s.views.items()} == views0
    for reps in (1, 2):
        s.replay(reps)
        s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, u0, 4 * steps, 0.25)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


def test_partially_pinned_input_is_bounced_through_a_copy(fake, monkeypatch):
    """A host input registered over fewer rows than a view uploads (the
    bench pins each rank's rows; a fused chain's view is KL rows deeper) must
    go through a fresh copy: a DMA straddling a registration edge is invalid,
    and np.ascontiguousarray of a contiguous slice would alias the input."""
    lib = fake(1)
    seen = []
    orig = type(lib).cq_copy_box_h2d

    def spy(self, d, s, eb, dst, host, halloc, box):
        seen.append(getattr(host, "value", host))
        return orig(self, d, s, eb, dst, host, halloc, box)
    monkeypatch.setattr(type(lib), "cq_copy_box_h2d", spy)
    monkeypatch.setattr(E, "_pin_state", lambda start, end: "partial")
    h, w = 64, 32
    u0 = np.random.default_rng(1).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=2, kind="float32", u0=u0, up0=u0)
    res = E.run(cq.generate_commands(prog.graph(), 1), placement=E.Placement(1, 0, (0,)))
    base, end = u0.ctypes.data, u0.ctypes.data + u0.nbytes
    assert seen and all(not (base <= p < end) for p in seen)
    from oracle import native as onat
    u, up = onat.wave_run(u0, u0, 2, 0.25)
    assert dsl.same_bits(res.buffers["u"], u)


def test_input_registrations_end_with_their_arrays(fake):
    """Page-locked input spans live as long as the arrays owning them:
    repeated runs over one input register it once, and dropping the program
    and its arrays unregisters it (no process-lifetime growth, run_batch over
    fresh per-job inputs included)."""
    import gc
    lib = fake(1)
    live = set()
    reg, unreg = lib.cq_host_register, lib.cq_host_unregister
    lib.cq_host_register = lambda p, n: live.add(_addr(p)) or reg(p, n)
    lib.cq_host_unregister = lambda p: live.discard(_addr(p)) or unreg(p)
    n = (E.PIN_MIN_BYTES // 8) + 1024
    x = np.random.default_rng(3).uniform(-1, 1, n)
    y = np.ones(n)
    prog = W.saxpy_program(n, kind="float64", x=x, y=y)
    plan = cq.generate_commands(prog.graph(), 2)
    E.run(plan, placement=E.Placement(1, 0, (0,)), trace=False)
    kept = dict(E._pinned)
    assert len(kept) == 2 and live == {s for s, _e in kept}   # x and y; the result's span was temporary
    E.run(plan, placement=E.Placement(1, 0, (0,)), trace=False)
    assert E._pinned == kept                                   # registered once
    jobs = [({"x": np.full(n, float(k)), "y": y}, None) for k in range(3)]
    E.run_batch(plan, jobs, placement=E.Placement(1, 0, (0,)))
    del jobs
    gc.collect()
    assert E._pinned == kept and live == {s for s, _e in kept}, "fresh per-job inputs must not stay registered"
    del prog, plan, x, y, kept
    gc.collect()
    assert not E._pinned and not live


def _addr(p):
    return p.value if hasattr(p, "value") else int(p)


def test_fused_wave_chain_float64(fake):
    """float64 (the reference's own kind) chains fuse too, with the same
    8/4-step block planning as float32."""
    from oracle import native as onat
    fake(1)
    h, w, steps = 160, 48, 22
    u0 = np.random.default_rng(31).uniform(0, 1, (h, w))
    prog = W.wave_program(h, w, steps=steps, kind="float64", c=0.3, u0=u0, up0=u0)
    s = E.Session(cq.generate_commands(prog.graph(), 2), E.Placement(1, 0, (0,)))
    ch = s.chains[0]
    assert [b.kl for b in ch.blocks] == [4, 8, 8] and len(ch.plain) == 2
    s.execute(upload=True)
    s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, u0, steps, 0.3)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


def test_run_temporaries_are_freed_by_recycle(fake):
    """An in-place stencil (a read at a non-zero offset of the buffer the
    task writes) snapshots its read region into a run temporary; repeated
    runs of one session free them at recycle instead of accumulating."""
    lib = fake(1)
    ext = cq.Box.from_shape((64,))
    bufs = {"a": cq.Buffer("a", ext, "float32", cq.BufferInit.iota())}
    body = {"a": cq.parse_kernel("ar[i-1] + ar[i+1]", {"ar": 1}, set(), 1)}
    t = cq.Task("relax", ext, [cq.Accessor("a", cq.AccessMode.READ, cq.Neighborhood((1,)), name="ar"),
                               cq.Accessor("a", cq.AccessMode.WRITE)], body)
    g = cq.TaskGraph(bufs)
    g.submit(t)
    s = E.Session(cq.generate_commands(g, 1), E.Placement(1, 0, (0,)))
    live = []
    for _ in range(4):
        s.execute(upload=True)
        s.synchronize()
        res = s.results()
        assert s.scratch   # the snapshot
        s.recycle()
        assert not s.scratch
        live.append(len(lib.blocks))
    s.close()
    a = np.arange(64, dtype=np.float32)
    want = np.concatenate([[a[0] + a[1]], a[:-2] + a[2:], [a[-2] + a[-1]]]).astype(np.float32)
    assert dsl.same_bits(res["a"], want)
    assert live[1] == live[-1], live


def test_run_batch_raises_posted_error_flag(fake):
    """run_batch reads each run's error flag from a copy posted behind its
    read-back and raises the reference's exception, also for the last runs
    (which are only drained, never recycled)."""
    lib = fake(1)
    prog = W.saxpy_program(64, kind="float32")
    plan = cq.generate_commands(prog.graph(), 2)
    lib.flag = N.CQ_ERR_EVAL
    with pytest.raises(cq.EvalError):
        E.run_batch(plan, [(None, None)] * 2, placement=E.Placement(1, 0, (0,)))
    lib.flag = None
    assert len(E.run_batch(plan, [(None, None)] * 3, placement=E.Placement(1, 0, (0,)))) == 3


def test_run_batch_matches_run(fake):
    """run_batch (two sessions in flight, their own upload / read-back
    streams) returns, per job, exactly what run() returns -- including jobs
    with their own input arrays."""
    from oracle import native as onat
    fake(1)
    h, w, steps = 96, 32, 10
    u0 = np.random.default_rng(51).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), 2)
    other = np.random.default_rng(52).uniform(0, 1, (h, w)).astype(np.float32)
    jobs = [(None, None), ({"u": other, "up": other}, None), (None, None), (None, None)]
    res = E.run_batch(plan, jobs, placement=E.Placement(1, 0, (0,)))
    for (inp, _o), r in zip(jobs, res):
        src = u0 if inp is None else other
        u, up = onat.wave_run(src, src, steps, 0.25)
        assert dsl.same_bits(r["u"], u) and dsl.same_bits(r["up"], up)


def test_shared_host_input_crosses_pcie_once(fake):
    """Buffers initialised from the same host array (a wave's u0 and
    up0 = u0) are uploaded once and copied device to device -- also on
    several nodes, where u's box (slab + halo rows) contains up's; results
    are unchanged, and distinct arrays are both uploaded."""
    from oracle import native as onat
    fake(1)
    h, w = 64, 48
    u0 = np.random.default_rng(5).uniform(0, 1, (h, w)).astype(np.float32)
    for nodes in (1, 2, 4):
        # each node uploads u over its slab plus its halo rows; up (same
        # host bytes, no halo -- or one halo row where the node's up view
        # holds one) is a device copy out of it
        moved = None
        for same in (True, False):
            up0 = u0 if same else u0.copy()
            prog = W.wave_program(h, w, steps=3, kind="float32", u0=u0, up0=up0)
            before = dict(E.STATS)
            res = E.run(cq.generate_commands(prog.graph(), nodes), placement=E.Placement(1, 0, (0,)))
            up_bytes = E.STATS["h2d_bytes"] - before["h2d_bytes"]
            dedup = E.STATS["upload_dedup_bytes"] - before["upload_dedup_bytes"]
            if same:
                assert up_bytes == (h + 2 * (nodes - 1)) * w * 4 and dedup >= h * w * 4, (nodes, up_bytes, dedup)
                moved = up_bytes + dedup
            else:   # distinct arrays: everything crosses PCIe
                assert up_bytes == moved and dedup == 0, (nodes, up_bytes, dedup)
            u, up = onat.wave_run(u0, up0, 3, 0.25)
            assert dsl.same_bits(res.buffers["u"], u) and dsl.same_bits(res.buffers["up"], up)


# ------------------------------------------------------- 8 ranks over gloo

def _rank8_main(rank, world, port, outdir):
    """The bench's shapes at 8 ranks (the driver's largest scaling point):
    a fused wave chain over 8 row slabs (KL-row exchanges between every
    neighbour pair, weak-scaled rows like bench.py) and the N-body 'all'
    mapper as one all-gather across the 8 ranks."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = FakeLib(1, GlooTransport())
    N._lib = lib
    pl = E.Placement(world, rank, (0,))
    results = {}
    u0 = np.random.default_rng(12).uniform(0, 1, (40 * world, 16)).astype(np.float32)
    prog = W.wave_program(40 * world, 16, steps=12, kind="float32", u0=u0, up0=u0)
    sess = E.Session(cq.generate_commands(prog.graph(), world), pl)
    assert [b.kl for b in sess.chains[0].blocks] == [4, 8]
    sess.execute(upload=True)
    sess.synchronize()
    res = sess.results()
    sess.close()
    if rank == 0:
        results["u"], results["up"] = res["u"], res["up"]
    pos, vel = W.nbody_inputs(8 * world)
    before = len(lib.launches)
    res = E.run(cq.generate_commands(W.nbody_program(8 * world, steps=2, pos=pos, vel=vel).graph(), world),
                placement=pl)
    results[f"allgathers_r{rank}"] = np.array(
        [sum(1 for x in lib.launches[before:] if isinstance(x, tuple) and x[0] == "allgather")])
    if rank == 0:
        results["P"], results["V"] = res.buffers["P"], res.buffers["V"]
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **results)
    dist.barrier()
    dist.destroy_process_group()


def test_eight_ranks_gloo(tmp_path):
    import torch.multiprocessing as mp
    from oracle import native as onat
    world = 8
    mp.start_processes(_rank8_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    r = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(world)]
    u0 = np.random.default_rng(12).uniform(0, 1, (40 * world, 16)).astype(np.float32)
    u, up = onat.wave_run(u0, u0, 12, 0.25)
    assert dsl.same_bits(r[0]["u"], u) and dsl.same_bits(r[0]["up"], up)
    assert all(int(x[f"allgathers_r{k}"][0]) == 1 for k, x in enumerate(r))
    pos, vel = W.nbody_inputs(8 * world)
    N._lib = FakeLib(1, LocalTransport())
    single = E.run(cq.generate_commands(W.nbody_program(8 * world, steps=2, pos=pos, vel=vel).graph(), 1),
                   placement=E.Placement(1, 0, (0,)))
    N._lib = None
    assert dsl.same_bits(r[0]["P"], single.buffers["P"]) and dsl.same_bits(r[0]["V"], single.buffers["V"])


# ------------------------------------------------- broadcast over 3 ranks

def _rank_bcast_main(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = FakeLib(1, GlooTransport())
    N._lib = lib
    plan = cq.generate_commands(W.row_broadcast_program(4 * world).graph(), world)
    res = E.run(plan, placement=E.Placement(world, rank, (0,)))
    # the byte all-gather the peer-memory setup uses (one NCCL all-gather)
    sess = E.Session(plan, E.Placement(world, rank, (0,)))
    blobs = sess.allgather_bytes(bytes([rank]) * 64)
    sess.close()
    assert blobs == [bytes([k]) * 64 for k in range(world)]
    n_b = sum(1 for x in lib.launches if isinstance(x, tuple) and x[0] == "bcast")
    n_g = sum(1 for x in lib.launches if isinstance(x, tuple) and x[0] == "group")
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), d=res.buffers.get("d", np.zeros(0)), n=np.array([n_b, n_g]))
    dist.barrier()
    dist.destroy_process_group()


def test_single_source_push_group_is_one_broadcast(tmp_path):
    """A push group sending one node's rows of a buffer to every other node
    is lowered to one in-place ncclBroadcast (cq_nccl_bcast) on every rank,
    with the same results as one process."""
    import torch.multiprocessing as mp
    world = 3
    mp.start_processes(_rank_bcast_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    r = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(world)]
    R, C = 4 * world, 64
    want = ((2 * np.arange(C, dtype=np.float32) + 1) * 3)[None, :] + np.arange(R, dtype=np.float32)[:, None]
    assert np.array_equal(r[0]["d"], want)
    for k in range(world):
        assert int(r[k]["n"][0]) == 1, r[k]["n"]   # one broadcast, no send/recv group for it
