"""The native C++ planner (csrc/cq_plan.cpp) emits the same Plan as the
Python planner and the reference -- ids, deps, regions (box decomposition
included), versions, push sources, frequencies, final locations.  Host-only:
runs without a GPU."""

import hashlib
import json
import os
import random

import pytest

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import workloads as W
from paper_2505_06022_b200.planner_native import generate_commands_native
from paper_2505_06022_b200.scheduler import generate_commands_py
from progjson import graph_of, program_from_json
from refcompat import plan_signature

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "programs.json")) as fh:
    PROGRAMS = json.load(fh)


@pytest.mark.parametrize("idx", range(len(PROGRAMS)))
def test_golden_programs(idx):
    entry = PROGRAMS[idx]
    buffers, tasks = program_from_json(entry["program"])
    g = graph_of(buffers, tasks)
    if entry.get("plan_sha") is None:
        with pytest.raises(cq.UninitializedReadError):
            cq.generate_commands(g, entry["nodes"])  # native defers, Python raises
        return
    for nodes in sorted({entry["nodes"], 1, 5, 8}):
        native = generate_commands_native(g, nodes)
        py = generate_commands_py(g, nodes)
        assert plan_signature(native) == plan_signature(py)
        assert cq.export_command_graph(native) == cq.export_command_graph(py)
    sig = plan_signature(generate_commands_native(g, entry["nodes"]))
    assert hashlib.sha256(sig.encode()).hexdigest() == entry["plan_sha"]


@pytest.mark.parametrize("builder", [
    lambda: W.saxpy_program(1 << 24, kind="float64"),
    lambda: W.wave_program(512, 256, steps=6, kind="float64"),
    lambda: W.nbody_program(4096, steps=2),
    lambda: W.sgemm_program(256, 256, 256),
])
def test_baseline_programs(builder):
    g = builder().graph()
    for nodes in (1, 2, 3, 4, 8):
        assert plan_signature(generate_commands_native(g, nodes)) == plan_signature(generate_commands_py(g, nodes))


def test_energy_targets_and_devices():
    g = W.saxpy_program(1000, kind="float64").graph()
    devs = [cq.DeviceModel(levels_ghz=(0.8, 1.0, 1.6), p_static_w=5.0 + i) for i in range(3)]
    for target in cq.EnergyTarget:
        a = generate_commands_native(g, 3, devices=devs, queue_target=target)
        b = generate_commands_py(g, 3, devices=devs, queue_target=target)
        assert plan_signature(a) == plan_signature(b)


@pytest.mark.reference
def test_reference_random_workloads():
    from refcompat import ref, ref_helpers, to_mine
    r = ref()
    rng = random.Random(4242)
    for _ in range(60):
        rbufs, rtasks = ref_helpers().random_workload(rng)
        rg = r.TaskGraph(rbufs)
        for t in rtasks:
            rg.submit(t)
        mg = cq.TaskGraph(to_mine(rbufs))
        for t in rtasks:
            mg.submit(to_mine(t))
        for nodes in (1, 2, 3, 4, 7):
            try:
                rplan = r.generate_commands(rg, nodes)
            except r.ClusterqError:
                with pytest.raises(cq.ClusterqError):
                    cq.generate_commands(mg, nodes)
                continue
            assert plan_signature(generate_commands_native(mg, nodes)) == plan_signature(rplan)
