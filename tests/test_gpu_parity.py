"""GPU parity: the B200 executor against the reference's own outputs (golden
fixtures) and the pinned CPU oracle.  Runs on a B200 via gpurun; every call
goes through the product path (executor -> ctypes -> libcq.so)."""

import json
import os

import numpy as np
import pytest

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import lowering, workloads as W
from paper_2505_06022_b200 import executor as E
from paper_2505_06022_b200.executor import run
from oracle import dsl
from oracle import native as onat
from progjson import graph_of, load_arrays, program_from_json

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "programs.json")) as fh:
    PROGRAMS = json.load(fh)
EXPECTED = load_arrays(os.path.join(GOLD, "expected.npz"))


def _run_program(buffers, tasks, nodes, **kw):
    plan = cq.generate_commands(graph_of(buffers, tasks), nodes)
    return run(plan, **kw)


@pytest.mark.parametrize("idx", range(len(PROGRAMS)))
def test_reference_programs_bit_exact(idx):
    """Every golden program (reference random workloads, bundled scenarios,
    wave ping-pong, SAXPY) at its node count and at 1 and 5 nodes reproduces
    the reference simulator's final buffers bit for bit."""
    entry = PROGRAMS[idx]
    for nodes in sorted({entry["nodes"], 1, 5}):
        buffers, tasks = program_from_json(entry["program"])
        if entry["error"] is not None:
            with pytest.raises(cq.ClusterqError) as info:
                _run_program(buffers, tasks, nodes)
            assert type(info.value).__name__ == entry["error"]
            return
        res = _run_program(buffers, tasks, nodes)
        for name in buffers:
            assert dsl.same_bits(res.buffers[name], EXPECTED[f"p{idx}__{name}"]), \
                (entry["name"], nodes, name)
        n_exec = sum(1 for e in res.trace if e.kind == "execute")
        assert n_exec == len(res.plan.executes())


@pytest.mark.parametrize("idx", [i for i, e in enumerate(PROGRAMS) if e["error"] is None][::4])
def test_interpreter_matches_fast_paths(idx, monkeypatch):
    entry = PROGRAMS[idx]
    monkeypatch.setattr(lowering, "FAST_PATHS", False)
    buffers, tasks = program_from_json(entry["program"])
    res = _run_program(buffers, tasks, entry["nodes"])
    for name in buffers:
        assert dsl.same_bits(res.buffers[name], EXPECTED[f"p{idx}__{name}"])


@pytest.mark.parametrize("idx", [i for i, e in enumerate(PROGRAMS) if e["error"] is None])
def test_jit_kernels_bit_exact(idx, monkeypatch):
    """DSL->CUDA JIT (NVRTC, sm_100a) for every launch, fast paths off:
    still the reference's bits."""
    from paper_2505_06022_b200 import jit
    monkeypatch.setattr(lowering, "FAST_PATHS", False)
    monkeypatch.setattr(jit, "MODE", "1")
    entry = PROGRAMS[idx]
    buffers, tasks = program_from_json(entry["program"])
    res = _run_program(buffers, tasks, entry["nodes"])
    for name in buffers:
        assert dsl.same_bits(res.buffers[name], EXPECTED[f"p{idx}__{name}"])


def test_jit_wave_large_matches_fast_path(monkeypatch):
    """A 2-D stencil body the fast path does not know (reordered terms) runs
    through the JIT at a size where it matters; compared with the oracle
    restatement of the same tree."""
    h, w = 2048, 2048
    u0 = np.random.default_rng(6).uniform(0, 1, (h, w)).astype(np.float32)
    body = ("u[i.0, i.1+1] + u[i.0, i.1-1] + u[i.0+1, i.1] + u[i.0-1, i.1] - 4 * u[i.0, i.1]")
    ext = cq.Box.from_shape((h, w))
    bufs = {"a": cq.Buffer("a", ext, "float32", cq.BufferInit.array(u0)),
            "b": cq.Buffer("b", ext, "float32", cq.BufferInit.zeros())}
    t = cq.Task("lap", ext, [cq.Accessor("a", cq.AccessMode.READ, cq.Neighborhood((1, 1)), name="u"),
                             cq.Accessor("b", cq.AccessMode.WRITE)],
                {"b": cq.parse_kernel(body, {"u": 2}, set(), 2)})
    res = _run_program(bufs, [t], 2)
    want = dsl.run_serial(bufs, [t])["b"]
    assert dsl.same_bits(res.buffers["b"], want)


@pytest.mark.parametrize("nodes", [1, 3, 4])
def test_saxpy_f32_bit_exact(nodes):
    n = (1 << 20) + 3
    x, y = W.saxpy_inputs(n, "float32", seed=0)
    prog = W.saxpy_program(n, alpha=2.0, kind="float32", x=x, y=y)
    res = run(cq.generate_commands(prog.graph(), nodes))
    assert dsl.same_bits(res.buffers["z"], onat.saxpy(2.0, x, y))


def test_saxpy_baseline_config_reference_inputs():
    """BASELINE config 1: N = 2^24, 4 chunks, x = iota, y = 1, alpha = 2:
    z = fl32(2i + 1) exactly."""
    n = 1 << 24
    prog = W.saxpy_program(n, kind="float32")
    res = run(cq.generate_commands(prog.graph(), 4))
    want = (2.0 * np.arange(n, dtype=np.float64) + 1.0).astype(np.float32)
    assert dsl.same_bits(res.buffers["z"], want)


@pytest.mark.parametrize("nodes", [1, 2, 3])
@pytest.mark.parametrize("kind", ["float32", "float64"])
def test_wave_bit_exact_vs_oracle(nodes, kind):
    h, w, steps = 257, 320, 7
    dt = np.float32 if kind == "float32" else np.float64
    u0 = np.random.default_rng(2).uniform(0, 1, (h, w)).astype(dt)
    up0 = np.random.default_rng(5).uniform(0, 1, (h, w)).astype(dt)
    prog = W.wave_program(h, w, steps=steps, kind=kind, c=0.25, u0=u0, up0=up0)
    res = run(cq.generate_commands(prog.graph(), nodes))
    u, up = onat.wave_run(u0, up0, steps, 0.25)
    assert dsl.same_bits(res.buffers["u"], u)
    assert dsl.same_bits(res.buffers["up"], up)


@pytest.mark.parametrize("nodes,steps,c", [(1, 22, 0.25), (1, 100, 0.25), (3, 22, 0.3), (4, 36, 0.3),
                                           (2, 9, 0.25), (1, 26, 0.1)])
def test_fused_wave_chain_bit_exact_vs_oracle(nodes, steps, c):
    """Temporal blocking (cq_wave5_fused: a KL=4 quarter block, then KL=8
    blocks, KL-row halo exchange between slabs, plain leftovers) reproduces
    the per-step oracle bit for bit -- also for a c whose products round
    (c = 0.3, 0.1) and subnormal neighbourhoods, where an FMA contraction of
    c*lap + (2u - upr) would differ."""
    from paper_2505_06022_b200.executor import Placement, Session
    h, w = 515, 640
    u0 = np.random.default_rng(21).uniform(0, 1, (h, w)).astype(np.float32)
    up0 = np.random.default_rng(22).uniform(0, 1, (h, w)).astype(np.float32)
    u0[:, :9] *= np.float32(1e-37)
    prog = W.wave_program(h, w, steps=steps, kind="float32", c=c, u0=u0, up0=up0)
    s = Session(cq.generate_commands(prog.graph(), nodes), Placement(1, 0, (0,)))
    assert len(s.chains) == 1
    s.execute(upload=True)
    s.synchronize()
    res = s.results()
    kinds = {k for k, *_ in s.launch_log}
    s.close()
    assert any(k.startswith("wave5_fused") for k in kinds)
    u, up = onat.wave_run(u0, up0, steps, c)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


@pytest.mark.parametrize("layout", [{"CQ_FUSED_ROWS": "7"}, {"CQ_FUSED_ROWS": "100"},
                                    {"CQ_FUSED_ROWS": "3000", "CQ_FUSED_MAP": "0"},
                                    {"CQ_FUSED_MAP": "1", "CQ_FUSED_WPB": "12"},
                                    {"CQ_FUSED_ROWS": "64", "CQ_FUSED_MAP": "2", "CQ_FUSED_WPB": "12"}])
def test_fused_wave_piece_layouts_bit_exact(layout, monkeypatch):
    """Every piece layout of the fused pass (rows per warp piece that split
    strips unevenly or cross strip ends, strip-major or strip-minor maps,
    12-warp blocks) gives the per-step oracle's bits, FMA-form blocks and
    slab edges included."""
    from paper_2505_06022_b200.executor import Placement, Session
    for k, v in layout.items():
        monkeypatch.setenv(k, v)
    h, w = 700, 1792
    u0 = np.random.default_rng(23).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=20, kind="float32", c=0.3, u0=u0, up0=u0)
    s = Session(cq.generate_commands(prog.graph(), 3), Placement(1, 0, (0,)))
    assert [b.kl for b in s.chains[0].blocks] == [4, 8, 8]
    s.execute(upload=True)
    s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, u0, 20, 0.3)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


@pytest.mark.parametrize("nodes,steps,w", [(1, 22, 384), (3, 16, 384), (1, 22, 1280), (3, 16, 1280)])
def test_fused_wave_chain_float64_bit_exact(nodes, steps, w):
    """The float64 fused kernel (two doubles per lane, scalar DADD/DMUL) is
    bit-identical to the float64 per-step oracle (w = 1280 has interior
    CTAs: 8 warps x 48 columns per block)."""
    from paper_2505_06022_b200.executor import Placement, Session
    h = 517
    u0 = np.random.default_rng(41).uniform(0, 1, (h, w))
    up0 = np.random.default_rng(42).uniform(0, 1, (h, w))
    u0[:, :5] *= 1e-300
    prog = W.wave_program(h, w, steps=steps, kind="float64", c=0.3, u0=u0, up0=up0)
    s = Session(cq.generate_commands(prog.graph(), nodes), Placement(1, 0, (0,)))
    assert s.chains
    s.execute(upload=True)
    s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, up0, steps, 0.3)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


def test_fused_wave_chain_huge_values_bit_exact():
    """Fields near the float32 range: the passes' magnitude bound is above
    the limit, so the fused kernel keeps the separate products (2u, 4u
    overflow in the tree where an FMA would not), and the result still equals
    the per-step oracle bit for bit."""
    from paper_2505_06022_b200.executor import Placement, Session
    h, w, steps = 515, 640, 12
    u0 = np.random.default_rng(24).uniform(0, 1, (h, w)).astype(np.float32)
    up0 = u0.copy()
    u0[200, 50:90] = np.float32(1.2e38)
    up0[300, 400:420] = np.float32(-9e37)
    prog = W.wave_program(h, w, steps=steps, kind="float32", c=0.3, u0=u0, up0=up0)
    s = Session(cq.generate_commands(prog.graph(), 2), Placement(1, 0, (0,)))
    assert s.chains
    s.execute(upload=True)
    s.synchronize()
    res = s.results()
    s.close()
    u, up = onat.wave_run(u0, up0, steps, 0.3)
    assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up)


@pytest.mark.parametrize("scale,c", [(1e30, 0.3), (1e-30, 0.25), (1.0, 0.45)])
def test_fused_wave_chain_fast_form_bit_exact(scale, c):
    """Blocks after the first take the FMA form of the body when the previous
    block's magnitude bound allows it (cq_wave5_fused_bounded); large, tiny
    and ordinary fields over many blocks stay bit-identical to the oracle."""
    from paper_2505_06022_b200.executor import Placement, Session
    # wide enough for interior CTAs (only those take the FMA form: a 12-warp
    # KL=8 block spans 12 x 112 columns plus halos)
    h, w, steps = 768, 3072, 64
    rng = np.random.default_rng(31)
    u0 = (rng.uniform(-1, 1, (h, w)) * scale).astype(np.float32)
    up0 = (rng.uniform(-1, 1, (h, w)) * scale).astype(np.float32)
    for nodes in (1, 3):
        prog = W.wave_program(h, w, steps=steps, kind="float32", c=c, u0=u0, up0=up0)
        s = Session(cq.generate_commands(prog.graph(), nodes), Placement(1, 0, (0,)))
        assert s.chains and len(s.chains[0].blocks) >= 6
        s.execute(upload=True)
        s.synchronize()
        res = s.results()
        s.close()
        u, up = onat.wave_run(u0, up0, steps, c)
        assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up), (scale, c, nodes)


@pytest.mark.parametrize("c", [0.3, -0.2, 0.25, 0.0])
def test_fused_wave_chain_fast_form_signed_zeros(c):
    """Fields of +0 / -0 and the smallest subnormals: exact cancellations
    (2u == p) and products underflowing to -0 must give the tree's signed
    zeros in the FMA form too (t = fma(2, u, -p), not -fma(-2, u, p); c*lap
    as fma(c, lap, +0), taken only for c > 0; c <= 0 keeps the exact form)."""
    from paper_2505_06022_b200.executor import Placement, Session
    h, w, steps = 768, 3072, 40   # interior CTAs exist (see above)
    rng = np.random.default_rng(33)
    vals = np.array([0.0, -0.0, 1e-45, -1e-45, 3e-45, -3e-45], dtype=np.float32)
    u0 = vals[rng.integers(0, len(vals), (h, w))]
    up0 = vals[rng.integers(0, len(vals), (h, w))]
    up0[::3] = u0[::3] * np.float32(2)   # exact cancellations 2u - p == 0
    for nodes in (1, 3):
        prog = W.wave_program(h, w, steps=steps, kind="float32", c=c, u0=u0, up0=up0)
        s_ = Session(cq.generate_commands(prog.graph(), nodes), Placement(1, 0, (0,)))
        assert s_.chains and len(s_.chains[0].blocks) >= 4
        s_.execute(upload=True)
        s_.synchronize()
        res = s_.results()
        s_.close()
        u, up = onat.wave_run(u0, up0, steps, c)
        assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up), (c, nodes)


def test_fused_wave_graph_replay_continues_the_simulation():
    """A captured fused execution replayed twice == two more plain fused
    executions == the 3x-longer simulation (the KL-row exchange makes a
    re-execution on resident data a true continuation; with an odd number of
    out-of-place blocks the capture holds two alternating graphs)."""
    from paper_2505_06022_b200.executor import Placement, Session
    h, w, steps = 384, 512, 26
    u0 = np.random.default_rng(23).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), 2)
    out = []
    for graph in (False, True):
        s = Session(plan, Placement(1, 0, (0,)))
        assert s.chains
        s.execute(upload=True)
        s.synchronize()
        s.recycle()
        if graph:
            s.capture()
            s.replay(2)
        else:
            for _ in range(2):
                s.execute(upload=False)
        s.synchronize()
        out.append(s.results())
        s.close()
    u, up = onat.wave_run(u0, u0, 3 * steps, 0.25)
    for o in out:
        assert dsl.same_bits(o["u"], u) and dsl.same_bits(o["up"], up)


def test_wave_unaligned_width_uses_generic_kernel():
    h, w = 64, 37
    u0 = np.random.default_rng(3).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=4, kind="float32", u0=u0, up0=u0)
    res = run(cq.generate_commands(prog.graph(), 3))
    u, up = onat.wave_run(u0, u0, 4, 0.25)
    assert dsl.same_bits(res.buffers["u"], u) and dsl.same_bits(res.buffers["up"], up)


@pytest.mark.parametrize("nodes", [1, 3])
def test_nbody_kick_within_tolerance(nodes):
    n, eps2, dt = 4096, 1e-2, 1e-3
    pos, vel = W.nbody_inputs(n)
    prog = W.nbody_program(n, steps=1, eps2=eps2, dt=dt, pos=pos, vel=vel)
    res = run(cq.generate_commands(prog.graph(), nodes))
    acc = onat.nbody_accel(pos, 0, n, eps2)
    got = res.buffers["V"][:, :3].astype(np.float64) / dt
    err = np.linalg.norm(got - acc, axis=1) / np.linalg.norm(acc, axis=1)
    assert err.max() <= 1e-4, err.max()
    want_pos = pos[:, :3].astype(np.float64) + dt * res.buffers["V"][:, :3]
    assert np.allclose(res.buffers["P"][:, :3], want_pos, rtol=0, atol=1e-6)
    assert np.array_equal(res.buffers["P"][:, 3], pos[:, 3])


def test_nbody_gpu_count_invariance():
    n = 2048
    pos, vel = W.nbody_inputs(n)
    outs = []
    for nodes in (1, 2, 4):
        prog = W.nbody_program(n, steps=2, pos=pos, vel=vel)
        outs.append(run(cq.generate_commands(prog.graph(), nodes)).buffers)
    for o in outs[1:]:
        assert dsl.same_bits(o["P"], outs[0]["P"]) and dsl.same_bits(o["V"], outs[0]["V"])


@pytest.mark.parametrize("variant", ["ffma", "3xtf32"])
@pytest.mark.parametrize("nodes", [1, 4])
def test_sgemm_within_tolerance(variant, nodes):
    m, n, k = 512, 384, 256
    a, b = W.sgemm_inputs(m, n, k)
    prog = W.sgemm_program(m, n, k, variant=variant, a=a, b=b)
    res = run(cq.generate_commands(prog.graph(), nodes))
    rows = np.arange(0, m, 7)
    c, cabs = onat.sgemm_rows(a, b, rows)
    err = np.abs(res.buffers["C"][rows] - c) / cabs
    assert err.max() <= 1e-6, err.max()


@pytest.mark.parametrize("shape", [(512, 384, 256), (256, 512, 1024), (1000, 768, 2048)])
def test_tf32_raw_a_is_its_own_hi_part(shape, monkeypatch):
    """3xTF32 with A itself as the hi operand (the MMA drops the low 13
    mantissa bits) gives the same C bits as the explicitly masked copy."""
    import ctypes
    import torch
    from paper_2505_06022_b200 import _native as N
    N.call("cq_init_device", 0)
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.rand((m, k), device="cuda", generator=g) * 2 - 1
    b = torch.rand((k, n), device="cuda", generator=g) * 2 - 1
    out = []
    for raw in ("1", "0"):
        monkeypatch.setenv("CQ_TF32_RAW_HI", raw)
        c = torch.full((m, n), float("nan"), device="cuda")
        torch.cuda.synchronize()
        N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), k, ctypes.c_void_p(b.data_ptr()), n,
               ctypes.c_void_p(c.data_ptr()), n, m, n, k)
        N.call("cq_stream_synchronize", 0, 0)
        out.append(c.cpu().numpy())
    assert dsl.same_bits(out[0], out[1])
    ref = a.double().cpu().numpy() @ b.double().cpu().numpy()
    cabs = np.abs(a.double().cpu().numpy()) @ np.abs(b.double().cpu().numpy())
    assert (np.abs(out[0] - ref) / cabs).max() <= 1e-6


@pytest.mark.parametrize("shape", [(512, 384, 256), (256, 1000, 1024), (1000, 768, 2048), (384, 260, 96)])
@pytest.mark.parametrize("ldb_pad", [0, 12, 3])
def test_tf32_mn_major_b_matches_transposed(shape, ldb_pad, monkeypatch):
    """The CTA-pair kernel reading B MN-major straight from [k, n] (B its own
    hi part, only B_lo split, untransposed) gives the same C bits as the
    transposed Bt_hi / Bt_lo path -- ragged n (260: a 4-column last box),
    n not a multiple of the 256-column tile, and a padded row pitch (a pitch
    of n + 3 is not 16-byte aligned: both calls take the transposed path)."""
    import ctypes
    import torch
    from paper_2505_06022_b200 import _native as N
    N.call("cq_init_device", 0)
    m, n, k = shape
    ldb = n + ldb_pad
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.rand((m, k), device="cuda", generator=g) * 2 - 1
    bfull = torch.rand((k, ldb), device="cuda", generator=g) * 2 - 1
    out = []
    for mnb in ("1", "0"):
        monkeypatch.setenv("CQ_TF32_MNB", mnb)
        c = torch.full((m, n), float("nan"), device="cuda")
        torch.cuda.synchronize()
        N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), k, ctypes.c_void_p(bfull.data_ptr()), ldb,
               ctypes.c_void_p(c.data_ptr()), n, m, n, k)
        N.call("cq_stream_synchronize", 0, 0)
        out.append(c.cpu().numpy())
    assert dsl.same_bits(out[0], out[1])
    an = a.double().cpu().numpy()
    bn = bfull[:, :n].double().cpu().numpy()
    ref = an @ bn
    cabs = np.abs(an) @ np.abs(bn)
    assert (np.abs(out[0] - ref) / cabs).max() <= 1e-6


def test_fused_pass_rejects_bad_arguments():
    """The C-ABI fails loudly (NativeError with the reason) on arguments the
    fused pass cannot honour, instead of computing something else."""
    import ctypes
    import torch
    from paper_2505_06022_b200 import _native as N
    N.call("cq_init_device", 0)
    h, w = 64, 256
    t = [torch.zeros((h, w), device="cuda") for _ in range(4)]

    def view(x):
        v = N.CqView()
        v.ptr = x.data_ptr()
        v.alloc = N.box3((0, 0), (h, w))
        v.stride[:] = [h * w, w, 1]
        return v
    vs = [view(x) for x in t]
    ext = N.box3((0, 0), (h, w))

    def call(levels=8, out=(0, h), views=vs, k2=2.0):
        N.call("cq_wave5_fused_bounded", 0, 0, N.CQ_F32, levels, ctypes.byref(views[0]), ctypes.byref(views[1]),
               ctypes.byref(views[2]), ctypes.byref(views[3]), 0, h, out[0], out[1], ctypes.byref(ext), 0.25,
               k2, 4.0, None, None)
    call()   # valid
    N.call("cq_stream_synchronize", 0, 0)
    with pytest.raises(cq.NativeError, match="levels"):
        call(levels=5)
    with pytest.raises(cq.NativeError, match="alias"):
        call(views=[vs[0], vs[1], vs[0], vs[3]])
    with pytest.raises(cq.NativeError, match="constants"):
        call(k2=3.0)


def test_integer_division_by_zero_raises_eval_error():
    ext = cq.Box.from_shape((16,))
    bufs = {"a": cq.Buffer("a", ext, "int64", cq.BufferInit.iota()),
            "b": cq.Buffer("b", ext, "int64", cq.BufferInit.zeros())}
    body = {"b": cq.parse_kernel("7 / (a[i] - 5)", {"a": 1}, set(), 1)}
    t = cq.Task("div", ext, [cq.Accessor("a", cq.AccessMode.READ), cq.Accessor("b", cq.AccessMode.WRITE)], body)
    with pytest.raises(cq.EvalError):
        _run_program(bufs, [t], 2)


@pytest.mark.parametrize("jobs", [1, 4])
def test_run_batch_reports_eval_error(jobs):
    """run_batch checks each run's error flag from a copy queued behind its
    read-back (no blocking read); the error surfaces for the last run too."""
    ext = cq.Box.from_shape((16,))
    bufs = {"a": cq.Buffer("a", ext, "int64", cq.BufferInit.iota()),
            "b": cq.Buffer("b", ext, "int64", cq.BufferInit.zeros())}
    body = {"b": cq.parse_kernel("7 / (a[i] - 5)", {"a": 1}, set(), 1)}
    t = cq.Task("div", ext, [cq.Accessor("a", cq.AccessMode.READ), cq.Accessor("b", cq.AccessMode.WRITE)], body)
    g = cq.TaskGraph(bufs)
    g.submit(t)
    plan = cq.generate_commands(g, 2)
    with pytest.raises(cq.EvalError):
        E.run_batch(plan, [(None, None)] * jobs, depth=2)
    # the flag was cleared: a clean program runs afterwards
    prog = W.saxpy_program(4099, kind="float32")
    E.run_batch(cq.generate_commands(prog.graph(), 2), [(None, None)] * 2)


def test_mapper_violation_raises():
    """A Fixed-mapped read whose clamped point leaves the declared region
    passes the static footprint check but fails at run time
    (ReadView.read, model.py:442-453)."""
    ext = cq.Box.from_shape((8,))
    bufs = {"a": cq.Buffer("a", ext, "float64", cq.BufferInit.iota()),
            "b": cq.Buffer("b", ext, "float64", cq.BufferInit.zeros())}
    fixed = cq.Fixed(cq.Region(1, [cq.Box((2,), (4,))]))
    body = {"b": cq.parse_kernel("a[i-3]", {"a": 1}, set(), 1)}
    t = cq.Task("bad", cq.Box.from_shape((2,)),
                [cq.Accessor("a", cq.AccessMode.READ, fixed), cq.Accessor("b", cq.AccessMode.WRITE)], body)
    with pytest.raises(cq.MapperViolationError):
        _run_program(bufs, [t], 1)


def test_trace_and_energy_accounting():
    prog = W.saxpy_program(1 << 20, kind="float32")
    plan = cq.generate_commands(prog.graph(), 4)
    res = run(plan, energy=True)
    kinds = [e.kind for e in res.trace]
    assert kinds.count("execute") == 4 and kinds.count("push") == kinds.count("await_push") == 6
    assert res.makespan > 0
    rep = cq.account_energy(res.trace, plan.devices, res.makespan)
    assert rep.total_kernel_energy + rep.total_idle_energy == rep.total_device_energy


def test_nbody_baseline_size_sampled():
    """BASELINE config 2 size: 262,144 bodies; 1,024 sampled i-bodies x all
    j against the float64 oracle (SURVEY.md §8d tolerance 1e-4), on 1 node
    and on 8 nodes sharing the GPU (the 'all' mapper's all-gather between
    them); the 8-node result is bit-identical to the 1-node one (fixed,
    GPU-count independent j order)."""
    n, eps2, dt = 262144, 1e-2, 1e-3
    pos, vel = W.nbody_inputs(n)
    prog = W.nbody_program(n, steps=1, eps2=eps2, dt=dt, pos=pos, vel=vel)
    idx = np.random.default_rng(0).choice(n, 1024, replace=False)
    want = onat.nbody_accel_idx(pos, idx, eps2)
    out = {}
    for nodes in (1, 8):
        res = run(cq.generate_commands(prog.graph(), nodes), trace=False)
        got = res.buffers["V"][idx, :3].astype(np.float64) / dt
        err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
        assert err.max() <= 1e-4, (nodes, err.max())
        out[nodes] = res.buffers
    for name in ("P", "V"):
        assert dsl.same_bits(out[1][name], out[8][name]), name


@pytest.mark.parametrize("variant", ["3xtf32", "ffma"])
def test_sgemm_baseline_size_sampled(variant):
    """BASELINE config 3 size: 16384^3 fp32 with slice mappers on 1 node and
    on 8 nodes (2048-row A / C slabs, B everywhere); 256 sampled rows of C
    against a float64 oracle, |C - C64| / sum|a||b| <= 1e-6."""
    m = 16384
    a, b = W.sgemm_inputs(m, m, m)
    prog = W.sgemm_program(m, m, m, variant=variant, a=a, b=b)
    rows = np.random.default_rng(1).choice(m, 256, replace=False)
    c, cabs = onat.sgemm_rows(a, b, rows)
    for nodes in (1, 8):
        res = run(cq.generate_commands(prog.graph(), nodes), trace=False)
        err = np.abs(res.buffers["C"][rows] - c) / cabs
        assert err.max() <= 1e-6, (nodes, err.max())
        del res


@pytest.mark.parametrize("nodes", [1, 3])
def test_graph_replay_equals_plain_replay(nodes):
    from paper_2505_06022_b200.executor import Placement, Session
    h, w = 256, 384
    u0 = np.random.default_rng(8).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=6, kind="float32", u0=u0, up0=u0)
    plan = cq.generate_commands(prog.graph(), nodes)
    out = []
    for graph in (False, True, "timed"):
        s = Session(plan, Placement(1, 0, (0,)))
        s.execute(upload=True)
        s.synchronize()
        s.recycle()
        if graph:
            s.capture(timed=graph == "timed")
            s.replay(3)
        else:
            for _ in range(3):
                s.execute(upload=False)
        s.synchronize()
        if graph == "timed":
            # one (start, stop) pair of event-record nodes per launch, re-taken per replay
            waves = [x for x in s.graph_log if x[0] == "wave5"]
            assert len(waves) >= 6
            times = [s.elapsed_ms(a, b) for _k, _c, _d, _s, a, b in waves]
            assert all(0.0 < t < 1e3 for t in times)
        out.append(s.results())
        s.close()
    for o in out[1:]:
        assert dsl.same_bits(out[0]["u"], o["u"]) and dsl.same_bits(out[0]["up"], o["up"])


def test_run_batch_two_in_flight_matches_oracle():
    """run_batch (upload of job k+1 overlapping kernels and read-back of job
    k, separate copy streams per session) == the oracle per job."""
    from paper_2505_06022_b200.executor import run_batch
    h, w, steps = 515, 640, 22
    a = np.random.default_rng(61).uniform(0, 1, (h, w)).astype(np.float32)
    b = np.random.default_rng(62).uniform(0, 1, (h, w)).astype(np.float32)
    plan = cq.generate_commands(W.wave_program(h, w, steps=steps, kind="float32", u0=a, up0=a).graph(), 2)
    jobs = [(None, None), ({"u": b, "up": b}, None), (None, None), ({"u": b, "up": a}, None), (None, None)]
    res = run_batch(plan, jobs)
    for (inp, _o), r in zip(jobs, res):
        u0, up0 = (a, a) if inp is None else (inp["u"], inp["up"])
        u, up = onat.wave_run(u0, up0, steps, 0.25)
        assert dsl.same_bits(r["u"], u) and dsl.same_bits(r["up"], up)


def test_wave_baseline_size_bit_exact():
    """BASELINE config 1 at full size: 16384 x 16384 fp32, 100 steps,
    temporally blocked (1 four-step + 12 eight-step passes) on one GPU and
    on 4 and 8 nodes sharing it (KL-row halo exchanges between the slabs),
    against the OpenMP oracle of the per-step tree -- bit for bit."""
    from paper_2505_06022_b200.executor import Placement, Session
    n, steps = 16384, 100
    u0 = W.wave_pulse(n, n, "float32")
    u, up = onat.wave_run(u0, u0, steps, 0.25)
    for nodes in (1, 4, 8):
        prog = W.wave_program(n, n, steps=steps, kind="float32", c=0.25, u0=u0, up0=u0)
        s = Session(cq.generate_commands(prog.graph(), nodes), Placement(1, 0, (0,)), trace=False)
        assert [b.kl for b in s.chains[0].blocks] == [4] + [8] * 12
        s.execute(upload=True)
        s.synchronize()
        res = s.results()
        s.close()
        assert dsl.same_bits(res["u"], u) and dsl.same_bits(res["up"], up), nodes


def test_kernel_energy_consumption_from_nvml():
    """SYnergy hooks as readings: run(energy=True) reads
    the NVML energy counter around the run; kernel_energy_consumption of each
    task is its duration share of the device's joules above the idle
    baseline, device_energy_consumption the counter delta."""
    from paper_2505_06022_b200 import measure
    n = 262144
    pos, vel = W.nbody_inputs(n)
    prog = W.nbody_program(n, steps=6, pos=pos, vel=vel)
    res = run(cq.generate_commands(prog.graph(), 1), energy=True)
    dev_j = measure.device_energy_consumption(res)
    assert dev_j > 0 and res.measured["nvml"]["devices"][0]["idle_w"] > 0
    kicks = [t for t in prog.graph().tasks if t.name.startswith("kick")]
    per = [measure.kernel_energy_consumption(res, t.id) for t in kicks]
    assert all(j > 0 for j in per)
    rep = measure.measured_energy(res)
    assert float(rep.total_kernel_energy) <= dev_j + 1e-9
    assert abs(float(sum(d.energy_j for d in rep.per_device)) - dev_j) < 1e-6


def test_measured_device_from_nvml_plans_and_runs():
    """The measured-table policy on hardware: a wave task's (seconds, joules)
    per iteration measured with NVML at the running SM clock
    (synergy.kernel_energy; clocks are never changed on this pool) feeds a
    MeasuredDevice; both planners then label every execute with that clock,
    and the run's measured energy report covers every task."""
    from paper_2505_06022_b200 import measure, synergy as S
    from paper_2505_06022_b200.executor import Placement, Session
    from paper_2505_06022_b200.planner_native import generate_commands_native
    from paper_2505_06022_b200.scheduler import generate_commands_py
    n, steps = 4096, 16
    u0 = W.wave_pulse(n, n, "float32")
    prog = W.wave_program(n, n, steps=steps, kind="float32", c=0.25, u0=u0, up0=u0)
    s = Session(cq.generate_commands(prog.graph(), 1), Placement(1, 0, (0,)), trace=False)
    s.execute(upload=True)
    s.synchronize()
    s.recycle()
    s.capture()
    r = S.kernel_energy(lambda: s.replay(1), 0, seconds=0.5, sync=s.synchronize)
    s.close()
    assert r["j_per_call"] > 0 and r["sm_mhz"] > 0
    table = S.MeasuredKernel("*", {r["sm_mhz"]: (r["s_per_call"] / steps, r["j_per_call"] / steps)})
    dev = S.MeasuredDevice({"*": table})
    for gen in (generate_commands_py, generate_commands_native):
        plan = gen(prog.graph(), 1, devices=dev, queue_target=cq.EnergyTarget.MIN_EDP)
        assert {c.frequency_ghz for c in plan.executes()} == {r["sm_mhz"] / 1000.0}
    res = run(plan, energy=True)
    rep = measure.measured_energy(res)
    assert len(rep.per_task) == steps and float(rep.total_device_energy) > 0
