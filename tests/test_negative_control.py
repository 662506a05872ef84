"""Negative controls: the parity checks must FAIL when
the data path loses data.

* the reference's own plan checker (``check_plan``, pkg/tests/helpers.py:
  59-165) accepts the repo planner's plans, and rejects one with a dropped
  Push;
* executing a plan with a dropped Push, or a temporally blocked chain whose
  KL-row halo exchange loses a row (fusion.halo_pushes), gives results that
  differ from the oracle -- on the numpy libcq double here and on a B200
  (``-m gpu``) -- while the intact runs match it bit for bit."""

import dataclasses

import numpy as np
import pytest

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import _native as N
from paper_2505_06022_b200 import executor as E
from paper_2505_06022_b200 import fusion
from paper_2505_06022_b200 import workloads as W
from paper_2505_06022_b200.region import Box, Region
from oracle import dsl
from oracle import native as onat
from refcompat import drop_push, ref, ref_helpers, to_reference, to_reference_plan


def _wave(h, w, steps, kind="float32", seed=4):
    dt = np.float32 if kind == "float32" else np.float64
    u0 = np.random.default_rng(seed).uniform(0, 1, (h, w)).astype(dt)
    return W.wave_program(h, w, steps=steps, kind=kind, c=0.25, u0=u0, up0=u0), u0


def _halo_push(plan):
    """A steady-state halo Push (produced by an earlier execute)."""
    return next(c for c in plan.commands if type(c).__name__ == "PushCommand" and c.deps
                and c.buffer in ("u", "up"))


def _check(plan, prog):
    r = ref()
    rbufs, rtasks = to_reference(prog.buffers, prog.tasks)
    rg = r.TaskGraph(rbufs)
    for t in rtasks:
        rg.submit(t)
    ref_helpers().check_plan(to_reference_plan(plan, rg), rbufs)


@pytest.mark.reference
def test_check_plan_accepts_repo_plans_and_rejects_a_dropped_push():
    progs = [_wave(40, 24, 6, "float64")[0], W.nbody_program(64, steps=2), W.sgemm_program(32, 24, 16),
             W.saxpy_program(1000, kind="float64")]
    for prog in progs:
        for nodes in (1, 2, 3, 5, 8):
            _check(cq.generate_commands(prog.graph(), nodes), prog)
    prog = progs[0]
    plan = cq.generate_commands(prog.graph(), 4)
    with pytest.raises(AssertionError):
        _check(drop_push(plan, _halo_push(plan)), prog)


@pytest.fixture
def fake(monkeypatch):
    from fakecq import FakeLib, LocalTransport
    lib = FakeLib(1, LocalTransport())
    monkeypatch.setattr(N, "_lib", lib)
    E._pinned.clear()
    return lib


def _lossy_halo(monkeypatch, node_pair=None):
    """fusion.halo_pushes losing the row nearest the boundary of one
    transfer (the first one of the block)."""
    real = fusion.halo_pushes

    def lossy(chain, kl, itemsize):
        out = list(real(chain, kl, itemsize))
        p = out[0]
        box = p.region.boxes[0]
        lo, hi = box.mins[0], box.maxs[0]
        # keep the kl - 1 rows farthest from the receiving slab
        lo, hi = (lo + 1, hi) if p.dst < p.src else (lo, hi - 1)
        out[0] = dataclasses.replace(p, region=Region.from_box(Box((lo, 0), (hi, box.maxs[1]))))
        return out
    monkeypatch.setattr(fusion, "halo_pushes", lossy)


def _negative_controls(monkeypatch, placement=None):
    # (1) a dropped one-row halo push (per-step execution)
    monkeypatch.setenv("CQ_WAVE_FUSE", "0")
    prog, u0 = _wave(48, 32, 6)
    plan = cq.generate_commands(prog.graph(), 4)
    u, up = onat.wave_run(u0, u0, 6, 0.25)
    good = E.run(plan, placement=placement)
    assert dsl.same_bits(good.buffers["u"], u) and dsl.same_bits(good.buffers["up"], up)
    bad = E.run(drop_push(plan, _halo_push(plan)), placement=placement)
    assert not (dsl.same_bits(bad.buffers["u"], u) and dsl.same_bits(bad.buffers["up"], up))
    # (2) a temporally blocked chain whose halo exchange loses one row
    monkeypatch.delenv("CQ_WAVE_FUSE")
    prog, u0 = _wave(96, 64, 12)
    plan = cq.generate_commands(prog.graph(), 3)
    u, up = onat.wave_run(u0, u0, 12, 0.25)
    with E.Session(plan, placement) as s:
        assert s.chains, "the 12-step chain must be temporally blocked"
    good = E.run(plan, placement=placement)
    assert dsl.same_bits(good.buffers["u"], u) and dsl.same_bits(good.buffers["up"], up)
    _lossy_halo(monkeypatch)
    bad = E.run(plan, placement=placement)
    assert not (dsl.same_bits(bad.buffers["u"], u) and dsl.same_bits(bad.buffers["up"], up))


def test_lost_transfers_break_parity_cpu(fake, monkeypatch):
    _negative_controls(monkeypatch, E.Placement(1, 0, (0,)))


@pytest.mark.gpu
def test_lost_transfers_break_parity_gpu(monkeypatch):
    _negative_controls(monkeypatch, E.Placement(1, 0, (0,)))
