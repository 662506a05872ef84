"""Scenario documents and the clusterq-compatible CLI (scenario.py, cli.py)
against the reference (pkg/src/clusterq/scenario.py, cli.py): the same
documents parse to the same scenarios (compared through the serialised
form), malformed ones fail with the same ScenarioError text, and the CLI's
planning output (DOT) is byte-identical.  Runs go through the executor on
the numpy libcq double here and on a B200 with -m gpu."""

import json
import os

import numpy as np
import pytest

from paper_2505_06022_b200 import _native as N
from paper_2505_06022_b200 import cli
from paper_2505_06022_b200 import executor as E
from paper_2505_06022_b200 import scenario as S
from paper_2505_06022_b200.errors import ScenarioError
from refcompat import ref

REF_SCENARIOS = "/root/reference/pkg/src/clusterq/scenarios"


def _ref_scenario_mod():
    ref()
    import sys
    return sys.modules["clusterq.scenario"]


def _task(**kw):
    t = {"name": "t", "range": [4], "writes": ["x"], "body": "1.0"}
    t.update(kw)
    return {"buffers": [{"name": "x", "extent": [4]}], "tasks": [t]}


def _mapper_doc(m):
    return {"buffers": [{"name": "x", "extent": [4]}, {"name": "z", "extent": [4]}],
            "tasks": [{"name": "t", "range": [4], "reads": [{"buffer": "x", "mapper": m}], "writes": ["z"],
                       "body": "x[i]"}]}


MINIMAL = {"buffers": [{"name": "x", "extent": [4]}]}
BAD = [
    {"buffers": [{"extent": [4]}]}, {"bogus": 1}, {"nodes": "two"}, {"nodes": 0}, {"nodes": True},
    {"buffers": [{"name": "x", "extent": [4], "frob": 1}]}, {"buffers": [{"name": "x", "extent": []}]},
    {"buffers": [{"name": "x", "extent": [0]}]}, {"buffers": [{"name": "x", "extent": [1, 2, 3, 4]}]},
    {"buffers": [{"name": "x", "extent": [2]}, {"name": "x", "extent": [2]}]},
    {**MINIMAL, "device": {}, "devices": [{}]}, {**MINIMAL, "target": "MIN_EDP", "queue_target": "MIN_EDP"},
    {**MINIMAL, "target": "TURBO"}, {**MINIMAL, "devices": []}, {**MINIMAL, "device": {"levels_ghz": []}},
    {**MINIMAL, "device": {"f_ref_ghz": 3.0}}, {**MINIMAL, "device": {"volts": 1}},
    {**MINIMAL, "link": {"latency_s": -1}}, {**MINIMAL, "link": {"speed": 1}},
    _task(reads=["nope"]), _task(writes=["nope"]), _task(body="1 +"), _task(target="FAST"),
    _task(writes=["x", "x"]), _task(extra=1), _task(params={"a": "b"}), _task(beta="x"), _task(body=3),
    _task(body={"x": "y[i]"}), _task(range=[4, 4]), _task(reads="x"),
    {"buffers": [{"name": "x", "extent": [2], "init": "random"}]},
    {"buffers": [{"name": "x", "extent": [2], "init": {"kind": "fill"}}]},
    {"buffers": [{"name": "x", "extent": [2], "init": {"kind": "zeros", "value": 1}}]},
    {"buffers": [{"name": "x", "extent": [2], "init": {"kind": "constant"}}]},
    {"buffers": [{"name": "x", "extent": [2], "init": {"kind": "values", "values": ["a"]}}]},
    _mapper_doc("wide"), _mapper_doc({"kind": "sparse"}), _mapper_doc({"kind": "neighborhood"}),
    _mapper_doc({"kind": "fixed", "region": []}), _mapper_doc({"kind": "slice", "dim": 3}),
    _mapper_doc({"kind": "fixed", "region": [{"min": [0], "max": [5]}]}), _mapper_doc({"kind": "all", "x": 1}),
    _mapper_doc({"kind": "neighborhood", "radius": -1}),
    {**MINIMAL, "expectations": [{"buffer": "y", "values": [0, 0, 0, 0]}]},
    {**MINIMAL, "expectations": [{"buffer": "x", "values": [0, 0]}]}, [], {"buffers": {}},
]


@pytest.mark.reference
def test_malformed_documents_fail_like_the_reference():
    RS = _ref_scenario_mod()
    r = ref()
    rejected = 0
    for doc in BAD:
        try:
            theirs = RS.scenario_to_dict(RS.scenario_from_dict(doc))
        except r.ClusterqError as want:
            with pytest.raises(ScenarioError) as got:
                S.scenario_from_dict(doc)
            assert str(got.value) == str(want), doc
            rejected += 1
        else:   # the reference parser accepts it (checked at submit): so must this one
            assert S.scenario_to_dict(S.scenario_from_dict(doc)) == theirs, doc
    assert rejected >= 40
    # the one deliberate difference: float32 is a known element kind here
    with pytest.raises(ScenarioError, match=r"scenario\.buffers\[0\]: buffer 'x': unknown element kind 'complex'"):
        S.scenario_from_dict({"buffers": [{"name": "x", "extent": [2], "element_kind": "complex"}]})


@pytest.mark.reference
def test_documents_parse_like_the_reference():
    RS = _ref_scenario_mod()
    docs = []
    for name in sorted(os.listdir(REF_SCENARIOS)):
        with open(os.path.join(REF_SCENARIOS, name)) as fh:
            docs.append(json.load(fh))
    for name in ("saxpy", "stencil", "wave"):
        with open(S.bundled_scenario_path(name)) as fh:
            docs.append(json.load(fh))
    docs.append({"nodes": 2, "devices": [{"levels_ghz": [1, 2], "f_ref_ghz": 1}, {"p_static_w": 3}],
                 "link": {"latency_s": 2e-6}, "queue_target": "MIN_ENERGY",
                 "buffers": [{"name": "a", "extent": [3, 4], "element_kind": "int64", "init": {"kind": "values",
                                                                                            "values": list(range(12))}},
                             {"name": "b", "extent": [3, 4], "init": "uninitialized"}],
                 "tasks": [{"name": "m", "range": [3, 4], "beta": 0.5, "target": "MIN_EDP",
                            "reads": [{"buffer": "a", "name": "p", "mapper": {"kind": "slice", "dim": 1}},
                                      {"buffer": "a", "name": "q", "mapper": {"kind": "fixed", "region": [
                                          {"min": [0, 0], "max": [1, 4]}]}}],
                            "writes": [{"buffer": "b", "name": "o"}], "body": {"o": "p[i.0, i.1] * 2 + q[i.0, i.1]"}}]})
    for doc in docs:
        mine = S.scenario_to_dict(S.scenario_from_dict(doc))
        if all(b.get("element_kind") != "float32" for b in doc["buffers"]):   # the reference has no float32
            assert mine == RS.scenario_to_dict(RS.scenario_from_dict(doc))
        assert S.scenario_to_dict(S.scenario_from_dict(mine)) == mine   # a fixed point


@pytest.mark.reference
def test_graph_command_matches_reference_cli(tmp_path, capsys):
    import sys
    ref()
    rcli = sys.modules.get("clusterq.cli")
    if rcli is None:
        import importlib
        rcli = importlib.import_module("clusterq.cli")
    for name in sorted(os.listdir(REF_SCENARIOS)):
        path = os.path.join(REF_SCENARIOS, name)
        for kind in ("task", "command"):
            for nodes in ("1", "3"):
                a, b = tmp_path / f"mine_{name}.dot", tmp_path / f"ref_{name}.dot"
                assert cli.main(["graph", path, "--kind", kind, "--nodes", nodes, "--out", str(a)]) == 0
                assert rcli.main(["graph", path, "--kind", kind, "--nodes", nodes, "--out", str(b)]) == 0
                assert a.read_text() == b.read_text(), (name, kind, nodes)


def test_cli_usage_and_missing_files_exit_1(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["run"])
    assert e.value.code == 1
    assert cli.main(["run", str(tmp_path / "nope.json")]) == 1
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["validate", str(bad)]) == 2


@pytest.fixture
def fake(monkeypatch):
    from fakecq import FakeNvmlLib, LocalTransport
    lib = FakeNvmlLib(1, LocalTransport())
    monkeypatch.setattr(N, "_lib", lib)
    monkeypatch.setattr(E, "local_placement", lambda: E.Placement(1, 0, (0,)))
    E._pinned.clear()
    return lib


def test_cli_run_writes_reports_with_measured_energy(fake, tmp_path, capsys):
    out = tmp_path / "out"
    assert cli.main(["run", "saxpy", "--out", str(out), "--energy"]) == 0
    rep = json.loads((out / "report.json").read_text())
    assert list(rep)[:4] == ["makespan_s", "per_task", "per_device", "transfers"]
    m = rep["measured"]
    assert m["per_task"][0]["name"] == "saxpy" and m["per_task"][0]["energy_j"] >= 0
    z = json.loads((out / "buf_z.json").read_text())
    assert z["values"] == [3 * i + 0.5 for i in range(16)]
    assert json.loads((out / "trace.json").read_text())["traceEvents"]
    assert cli.main(["validate", "wave"]) == 0
    assert cli.main(["run", "stencil", "--nodes", "2", "--target", "MIN_ENERGY", "--out", str(out)]) == 0


def test_expectation_failure_exits_2(fake, tmp_path, capsys):
    doc = json.loads(open(S.bundled_scenario_path("saxpy")).read())
    doc["expectations"][0]["values"][3] = -1
    p = tmp_path / "s.json"
    p.write_text(json.dumps(doc))
    assert cli.main(["run", str(p), "--out", str(tmp_path / "o")]) == 2
    assert "differs from expectation at index (3,)" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_run_on_gpu_with_nvml_energy(tmp_path):
    out = tmp_path / "out"
    assert cli.main(["run", "wave", "--out", str(out), "--energy"]) == 0
    rep = json.loads((out / "report.json").read_text())
    assert "energy_j_device0" in rep["measured"] and len(rep["measured"]["per_task"]) == 12
    assert cli.main(["validate", "wave", "--nodes", "5"]) == 0
