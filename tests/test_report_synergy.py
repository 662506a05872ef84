"""report.json schema (reference cli.py:85-115) and the measured-table
frequency policy (reference selection rule, energy.py:93-106)."""

import json
from fractions import Fraction

import pytest

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import _native as N
from paper_2505_06022_b200 import executor as E
from paper_2505_06022_b200 import report, workloads as W
from paper_2505_06022_b200.synergy import MeasuredKernel, select_measured
from fakecq import FakeLib, LocalTransport


def test_report_keys_and_identities(monkeypatch, tmp_path):
    monkeypatch.setattr(N, "_lib", FakeLib(1, LocalTransport()))
    prog = W.saxpy_program(64, kind="float64")
    plan = cq.generate_commands(prog.graph(), 3)
    res = E.run(plan)
    rep = report.build_report(res)
    assert list(rep) == ["makespan_s", "per_task", "per_device", "transfers"]
    assert rep["transfers"] == {"count": len(plan.pushes()), "total_bytes": sum(p.bytes for p in plan.pushes())}
    assert [t["id"] for t in rep["per_task"]] == [1]
    assert set(rep["per_task"][0]["frequency_ghz_per_node"]) == {"0", "1", "2"}
    report.write_outputs(res, tmp_path)
    doc = json.loads((tmp_path / "buf_z.json").read_text())
    assert doc["values"] == [2.0 * i + 1 for i in range(64)]
    assert "traceEvents" in json.loads((tmp_path / "trace.json").read_text())


def test_select_measured_follows_reference_rule():
    k = MeasuredKernel("wave", {1000: (2.0, 100.0), 1500: (1.5, 120.0), 1965: (1.2, 150.0)})
    assert select_measured(k, cq.EnergyTarget.MAX_PERF) == 1965
    assert select_measured(k, cq.EnergyTarget.MIN_ENERGY) == 1000
    # E*t: 200, 180, 180 -> tie goes to the higher clock
    assert select_measured(k, cq.EnergyTarget.MIN_EDP) == 1965
    # E*t^2: 400, 270, 216
    assert select_measured(k, cq.EnergyTarget.MIN_ED2P) == 1965


def test_select_measured_matches_model_selection_on_model_points():
    """Fed the reference DeviceModel's own (t, E) per level, the measured
    policy picks what the reference's select_frequency picks."""
    from paper_2505_06022_b200.energy import _objective, exec_time
    dev = cq.DeviceModel()
    for beta in (0.0, 0.3, 1.0):
        for t_ref in (Fraction(1, 1000), Fraction(3)):
            pts = {}
            for f in dev.levels_ghz:
                t = exec_time(t_ref, beta, dev.f_ref_ghz, f)
                pts[int(f * 1000)] = (t, dev._power_exact(f) * t)
            k = MeasuredKernel("m", pts)
            for target in cq.EnergyTarget:
                want = cq.select_frequency(dev, target, t_ref, beta)
                assert select_measured(k, target) == int(want * 1000)


def test_sweep_fit_and_select_on_a_simulated_nvml_device(monkeypatch):
    """SYnergy sweep logic on CPU: three clocks (max, ~75 %, ~50 %) of the
    supported list, a compute-bound and a memory-bound 'kernel' (time ~ 1/f
    vs constant), the reference time model's beta fitted from the measured
    points, and the reference selection rule over them."""
    import time as _t
    from fakecq import FakeNvmlLib
    from paper_2505_06022_b200 import _native as N
    from paper_2505_06022_b200 import synergy as S
    from paper_2505_06022_b200.energy import EnergyTarget
    lib = FakeNvmlLib(1)
    monkeypatch.setattr(N, "_lib", lib)
    clocks = S.sweep_clocks(S.supported_sm_clocks(0))
    assert clocks == [1965, 1500, 990]
    compute = S.sweep("compute", lambda: _t.sleep(0.008 * 1965 / lib.mhz), 0, clocks, seconds=0.25)
    memory = S.sweep("memory", lambda: _t.sleep(0.008), 0, clocks, seconds=0.25)
    assert compute.levels() == memory.levels() == [990, 1500, 1965]
    assert lib.mhz == 1965  # clocks reset after the sweep
    assert abs(float(S.fit_beta(compute))) < 0.3 and abs(float(S.fit_beta(memory)) - 1) < 0.3
    # a memory-bound kernel saves energy at a low clock at no time cost
    assert S.select_measured(memory, EnergyTarget.MIN_ENERGY) == 990
    assert S.select_measured(memory, EnergyTarget.MAX_PERF) == 1965
    # without permission only the running clock is measured
    lib.allow_lock = False
    only = S.sweep("memory", lambda: _t.sleep(0.002), 0, clocks, seconds=0.05)
    assert only.levels() == [1965]


def test_bench_clock_sweep_leg_on_the_simulated_device(monkeypatch):
    """bench.py's SYnergy leg end to end on the CPU double: three clocks per
    kernel, beta and per-target selections reported; without
    CQ_ALLOW_CLOCK_LOCK it reports why it did not run."""
    import types
    import bench
    from fakecq import FakeNvmlLib
    from paper_2505_06022_b200 import _native as N
    from paper_2505_06022_b200 import executor as E
    lib = FakeNvmlLib(1)
    monkeypatch.setattr(N, "_lib", lib)
    args = types.SimpleNamespace(size=64, wave_steps=8, nbody=256)
    dist = types.SimpleNamespace(world=1, rank=0)
    pl = E.Placement(1, 0, (0,))
    monkeypatch.delenv("CQ_ALLOW_CLOCK_LOCK", raising=False)
    assert bench.clock_sweep(args, dist, pl).startswith("not run")
    monkeypatch.setenv("CQ_ALLOW_CLOCK_LOCK", "1")
    monkeypatch.setattr(bench, "SWEEP_SECONDS", 0.05)
    out = bench.clock_sweep(args, dist, pl)
    assert out["clocks_mhz"] == [1965, 1500, 990]
    for name in ("wave5_100_steps", "nbody_3_steps"):
        assert len(out[name]["points"]) == 3
        assert set(out[name]["selected_mhz"]) == {"MAX_PERF", "MIN_ENERGY", "MIN_EDP", "MIN_ED2P"}
        assert out[name]["selected_mhz"]["MAX_PERF"] == 1965


def test_bench_reference_arm_contract_line():
    """`bench.py --impl reference` (the CPU port of the path, no GPU) prints
    one JSON line with the contract's keys; W is raised to the minimum 3."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--size", "256",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["warmup"] >= 3 and d["steps"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    # the driver pairs the arms by metric / unit / higher_is_better: the b200
    # arm's line (headline_line) must carry the same strings and config
    import types
    sys.path.insert(0, root)
    import bench
    with open(os.path.join(root, "BASELINE.json")) as fh:
        assert d["metric"] == json.load(fh)["metric"] == bench.METRIC
    args = types.SimpleNamespace(size=256, steps=2, warmup=3, wave_steps=bench.WAVE_STEPS)
    wave = {"value": 1.0, "ms_per_step": 1.0, "plan_s": 0.0, "replay": "cuda_graph", "execution": "",
            "e2e": {}, "roofline": {}, "clocks": {}, "gpu_launches": 1, "energy": None}
    mine = bench.headline_line(args, 1, wave, None, None, None)
    for key in ("metric", "unit", "higher_is_better", "config", "scaling", "dtype", "n_gpus", "steps", "warmup"):
        assert mine[key] == d[key], key
    assert d["ms_per_step"] > 0 and "100 time steps per bench step" in d["config"]["workload"]


def test_measured_energy_apportions_nvml_joules():
    """measure.measured_energy: device joules = the NVML delta; idle joules =
    idle power x the window no execute covers; kernel joules split over the
    device's executes by duration (SYnergy kernel_energy_consumption /
    device_energy_consumption as readings)."""
    from fractions import Fraction as F
    from paper_2505_06022_b200 import measure
    from paper_2505_06022_b200.executor import RunResult, TraceEvent
    tr = [TraceEvent("execute", 0, 0, F(0), F(1, 10), frequency_ghz=2.0, task_id=0, task_name="a"),
          TraceEvent("execute", 1, 1, F(1, 20), F(1, 10), frequency_ghz=2.0, task_id=0, task_name="a"),
          TraceEvent("execute", 0, 2, F(2, 10), F(3, 10), frequency_ghz=2.0, task_id=1, task_name="b"),
          TraceEvent("push", 0, 3, F(1, 10), F(1, 100), bytes=8)]
    nv = {"devices": {0: {"energy_j": 120.0, "idle_w": 100.0, "window_s": 0.6}},
          "node_device": {0: 0, 1: 0}}
    res = RunResult(buffers={}, trace=tr, makespan=F(1, 2), plan=None, measured={"nvml": nv})
    rep = measure.measured_energy(res)
    # busy = union [0, 0.15) + [0.2, 0.5) = 0.45 s -> idle 0.15 s x 100 W = 15 J, kernels 105 J
    assert float(rep.total_kernel_energy) == pytest.approx(105)
    assert measure.kernel_energy_consumption(res, 1) == pytest.approx(105 * 0.3 / 0.5)
    assert measure.kernel_energy_consumption(res, 0) == pytest.approx(105 * 0.2 / 0.5)
    assert float(sum(d.energy_j for d in rep.per_device)) == pytest.approx(120)
    assert measure.device_energy_consumption(res) == 120.0
    with pytest.raises(cq.ValidationError):
        measure.measured_energy(RunResult({}, tr, F(1), None, {}))


def test_measured_device_drives_plan_frequencies():
    """A MeasuredDevice makes generate_commands pick each task's clock with
    select_measured over its kernel's table (both planners), and
    account_energy charges the measured power at that clock."""
    from fractions import Fraction as F
    from paper_2505_06022_b200 import synergy as S, workloads as W
    from paper_2505_06022_b200.planner_native import generate_commands_native
    from paper_2505_06022_b200.scheduler import generate_commands_py
    saxpy = S.MeasuredKernel("saxpy", {1965: (1.0, 10.0), 1500: (1.1, 8.0), 990: (1.5, 9.0)})
    other = S.MeasuredKernel("*", {1965: (1.0, 5.0), 1500: (1.3, 6.0), 990: (2.0, 7.0)})
    dev = S.MeasuredDevice({"saxpy": saxpy, "*": other})
    assert dev.levels_ghz == (0.99, 1.5, 1.965)
    prog = W.saxpy_program(4096, kind="float64")
    for target, want in ((cq.EnergyTarget.MIN_ENERGY, 1.5), (cq.EnergyTarget.MAX_PERF, 1.965),
                         (cq.EnergyTarget.MIN_EDP, 1.5), (cq.EnergyTarget.MIN_ED2P, 1.5)):
        for gen in (generate_commands_py, generate_commands_native):
            plan = gen(prog.graph(), 3, devices=dev, queue_target=target)
            assert {c.frequency_ghz for c in plan.executes()} == {want}, (target, gen)
    assert dev.power_watts(1.5) == pytest.approx(float((F(8) / F(11, 10) + F(6) / F(13, 10)) / 2))


def test_measured_energy_of_a_run_shorter_than_the_nvml_counter_step(monkeypatch):
    """NVML's energy counter advances in coarse steps: a run read between two
    plain counter reads can see no change.  run(energy=True) opens and closes
    its window on counter steps, so a short run still reports the joules of
    a window that covers it (the GPU failure of round 2: 0 J for 16 steps of a
    4096^2 wave)."""
    from fakecq import FakeNvmlLib, LocalTransport
    from paper_2505_06022_b200 import _native as N
    from paper_2505_06022_b200 import executor as E
    from paper_2505_06022_b200 import measure
    from paper_2505_06022_b200.workloads import saxpy_program
    lib = FakeNvmlLib(1, LocalTransport(), tick_s=0.05)
    monkeypatch.setattr(N, "_lib", lib)
    monkeypatch.setattr(E, "local_placement", lambda: E.Placement(1, 0, (0,)))
    E._pinned.clear()
    prog = saxpy_program(64, chunks=2)
    res = E.run(cq.generate_commands(prog.graph(), 1), energy=True)
    dev = res.measured["nvml"]["devices"][0]
    assert dev["window_s"] >= 0.04 and dev["energy_j"] > 0
    rep = measure.measured_energy(res)
    assert float(rep.total_device_energy) > 0 and len(rep.per_task) == 1
