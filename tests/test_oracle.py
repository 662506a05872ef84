"""Pin the CPU oracle against the reference before trusting it.

The golden fixtures were produced by the reference simulator itself
(tests/golden/make_golden.py); every oracle must reproduce them bit-exactly.
Where the reference is importable (this container) the oracle is also
checked against fresh reference runs."""

import json
import os
import random

import numpy as np
import pytest

from oracle import dsl
from oracle import native as onat
from progjson import load_arrays, program_from_json

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _programs():
    with open(os.path.join(GOLD, "programs.json")) as fh:
        return json.load(fh)


EXPECTED = load_arrays(os.path.join(GOLD, "expected.npz"))


@pytest.mark.parametrize("idx", range(len(_programs())))
def test_dsl_oracle_matches_reference_golden(idx):
    entry = _programs()[idx]
    buffers, tasks = program_from_json(entry["program"])
    if entry["error"] is not None:
        with pytest.raises(dsl.OracleError):
            dsl.run_serial(buffers, tasks)
        return
    out = dsl.run_serial(buffers, tasks)
    for name in buffers:
        key = f"p{idx}__{name}"
        assert dsl.same_bits(out[name], EXPECTED[key]), (entry["name"], name)


def test_c_oracle_wave_f64_matches_reference_golden():
    for idx, entry in enumerate(_programs()):
        if not entry["name"].startswith("wave_"):
            continue
        buffers, tasks = program_from_json(entry["program"])
        u0 = dsl.initial_array(buffers["u"])
        up0 = dsl.initial_array(buffers["up"])
        u, up = onat.wave_run(u0, up0, len(tasks), 0.25)
        assert dsl.same_bits(u, EXPECTED[f"p{idx}__u"])
        assert dsl.same_bits(up, EXPECTED[f"p{idx}__up"])


def test_c_oracle_saxpy_matches_reference_golden():
    idx = next(i for i, e in enumerate(_programs()) if e["name"] == "saxpy_4096")
    x = np.arange(4096, dtype=np.float64)
    y = np.ones(4096)
    assert dsl.same_bits(onat.saxpy(2.0, x, y), EXPECTED[f"p{idx}__z"])
    assert np.array_equal(EXPECTED[f"p{idx}__z"], 2 * x + 1)


def test_two_float32_restatements_agree():
    """The numpy (per-operator) and C (-ffp-contract=off) float32 wave steps
    are independent restatements; they must agree bit for bit."""
    from paper_2505_06022_b200 import workloads as W
    h, w = 37, 29
    u0 = np.random.default_rng(1).uniform(0, 1, (h, w)).astype(np.float32)
    up0 = np.random.default_rng(2).uniform(0, 1, (h, w)).astype(np.float32)
    prog = W.wave_program(h, w, steps=3, kind="float32", u0=u0, up0=up0)
    out = dsl.run_serial(prog.buffers, prog.tasks)
    u, up = onat.wave_run(u0, up0, 3, 0.25)
    assert dsl.same_bits(out["u"], u) and dsl.same_bits(out["up"], up)
    s = onat.saxpy(2.0, u0.ravel(), up0.ravel())
    sp = W.saxpy_program(h * w, kind="float32", x=u0.ravel(), y=up0.ravel())
    assert dsl.same_bits(dsl.run_serial(sp.buffers, sp.tasks)["z"], s)


def test_nbody_oracle_properties():
    """N-body has no reference arithmetic: check the oracle's
    physics instead -- momentum conservation (sum m_i a_i = 0) and an
    analytic two-body case."""
    from paper_2505_06022_b200 import workloads as W
    pos, _ = W.nbody_inputs(256)
    acc = onat.nbody_accel(pos, 0, 256, 1e-2)
    m = pos[:, 3].astype(np.float64)
    total = (m[:, None] * acc).sum(axis=0)
    assert np.abs(total).max() < 1e-9 * np.abs(m[:, None] * acc).sum()
    two = np.array([[0, 0, 0, 1], [1, 0, 0, 2]], np.float32)
    a = onat.nbody_accel(two, 0, 2, 1e-30)
    assert np.allclose(a[0], [2, 0, 0]) and np.allclose(a[1], [-1, 0, 0])


def test_sgemm_oracle_rows():
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (64, 48)).astype(np.float32)
    b = rng.uniform(-1, 1, (48, 40)).astype(np.float32)
    c, cabs = onat.sgemm_rows(a, b, [0, 5, 63])
    want = a.astype(np.float64)[[0, 5, 63]] @ b.astype(np.float64)
    assert np.allclose(c, want, rtol=0, atol=1e-12)
    assert np.all(cabs >= np.abs(c) - 1e-12)


@pytest.mark.reference
def test_dsl_oracle_matches_fresh_reference_runs():
    from refcompat import ref, ref_helpers, to_mine
    r = ref()
    rng = random.Random(211)
    for _ in range(30):
        rbufs, rtasks = ref_helpers().random_workload(rng)
        g = r.TaskGraph(rbufs)
        for t in rtasks:
            g.submit(t)
        try:
            res = r.run(r.generate_commands(g, 2))
        except r.ClusterqError:
            continue
        out = dsl.run_serial(to_mine(rbufs), [to_mine(t) for t in rtasks])
        for name, arr in res.buffers.items():
            assert dsl.same_bits(out[name], arr)
