"""Planner and energy parity against reference-generated fixtures (runs
without the reference, e.g. on the GPU box)."""

import hashlib
import json
import os
from fractions import Fraction

import pytest

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import workloads as W
from progjson import graph_of, program_from_json
from refcompat import plan_signature

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "programs.json")) as fh:
    PROGRAMS = json.load(fh)


@pytest.mark.parametrize("idx", range(len(PROGRAMS)))
def test_plan_signature_matches_reference(idx):
    entry = PROGRAMS[idx]
    if entry["error"] is not None and entry.get("plan_sha") is None:
        buffers, tasks = program_from_json(entry["program"])
        try:
            plan = cq.generate_commands(graph_of(buffers, tasks), entry["nodes"])
        except cq.UninitializedReadError:
            assert entry["error"] == "UninitializedReadError"
        return
    buffers, tasks = program_from_json(entry["program"])
    plan = cq.generate_commands(graph_of(buffers, tasks), entry["nodes"])
    sig = plan_signature(plan)
    assert hashlib.sha256(sig.encode()).hexdigest() == entry["plan_sha"], entry["name"]


@pytest.mark.parametrize("name,builder,nodes", [
    ("saxpy_2p24_n4", lambda: W.saxpy_program(1 << 24, kind="float64"), 4),
    ("wave_256x128_s4_n4", lambda: W.wave_program(256, 128, steps=4, kind="float64"), 4),
    ("nbody_1024_s2_n4", lambda: W.nbody_program(1024, steps=2), 4),
    ("sgemm_256_n8", lambda: W.sgemm_program(256, 256, 256), 8),
])
def test_baseline_dot_matches_reference(name, builder, nodes):
    with open(os.path.join(GOLD, "dot", name + ".dot")) as fh:
        want = fh.read()
    plan = cq.generate_commands(builder().graph(), nodes)
    assert cq.export_command_graph(plan) == want


def test_energy_selection_and_accounting_match_reference():
    with open(os.path.join(GOLD, "energy.json")) as fh:
        ref = json.load(fh)
    dev = cq.DeviceModel()
    for target, t_ref, beta, f in ref["selections"]:
        assert cq.select_frequency(dev, cq.EnergyTarget(target), Fraction(t_ref), beta) == f
    from paper_2505_06022_b200.executor import TraceEvent
    trace = [TraceEvent(k, n, c, Fraction(s), Fraction(d), frequency_ghz=f, task_id=t, task_name=tn)
             for k, n, c, s, d, f, t, tn in ref["trace"]]
    rep = cq.account_energy(trace, [dev] * 3, Fraction(ref["makespan"]))
    assert [[t.task_id, str(t.energy_j), str(t.duration_s)] for t in rep.per_task] == ref["per_task"]
    assert [[d.node, str(d.energy_j), str(d.busy_s), str(d.idle_s)] for d in rep.per_device] == \
        ref["per_device"]
    assert rep.total_kernel_energy + rep.total_idle_energy == rep.total_device_energy
