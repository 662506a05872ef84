"""Measured SYnergy energy: NVML joules behind the reference's energy hooks.

The reference charges model watts to logical time (energy.py:150-197).  A
B200 run with ``run(plan, energy=True)`` reads, per device, the idle power
before the run and the NVML energy counter at the counter step just before
the run and at the first step after it (``RunResult.measured["nvml"]``;
the counter advances in steps of tens of ms, so a window between two plain
reads can miss a short run entirely); ``measured_energy`` turns that into
the reference's ``EnergyReport``:

* device joules = the counter delta over the window between the two steps;
* idle joules = the pre-run idle power x the window time no execute covers
  (union of the device's execute intervals, CUDA-event times);
* kernel joules = device joules - idle joules, split over the device's
  execute events in proportion to their measured durations; a task's joules
  are the sum over its events -- ``kernel_energy_consumption(e)`` and
  ``device_energy_consumption()`` of the paper's SYnergy queue
   as readings, not a model.

The NVML counter advances in coarse steps, so per-task joules need runs of
tens of milliseconds or more; ``synergy.kernel_energy`` loops a single
kernel for >= 1 s when one kernel's J/iteration is wanted.
"""

from fractions import Fraction

from .energy import DeviceEnergy, EnergyReport, TaskEnergy
from .errors import ValidationError


def _union_length(intervals):
    total, end = Fraction(0), None
    for a, b in sorted(intervals):
        if end is None or a > end:
            total += b - a
            end = b
        elif b > end:
            total += b - end
            end = b
    return total


def measured_energy(result) -> EnergyReport:
    """EnergyReport of a run made with ``energy=True`` from NVML readings
    (see the module docstring); per_device is per plan node, a device's idle
    joules shared equally by the nodes it hosts."""
    nv = (result.measured or {}).get("nvml")
    if not nv:
        raise ValidationError("the run has no NVML readings (use run(..., energy=True))")
    node_dev = nv["node_device"]
    window = {d: Fraction(v["window_s"]) for d, v in nv["devices"].items()}
    events = [e for e in result.trace if e.kind == "execute"]
    by_dev = {}
    for e in events:
        by_dev.setdefault(node_dev[e.node], []).append(e)
    kernel_j, idle_j, busy_s = {}, {}, {}
    for d, v in nv["devices"].items():
        evs = by_dev.get(d, [])
        busy = _union_length([(Fraction(e.start), Fraction(e.start) + Fraction(e.duration)) for e in evs])
        busy = min(busy, window[d])
        idle = Fraction(v["idle_w"]) * (window[d] - busy)
        total = Fraction(v["energy_j"])
        idle_j[d] = min(idle, total)
        kernel_j[d] = total - idle_j[d]
        busy_s[d] = busy
    ev_j = {}
    for d, evs in by_dev.items():
        span = sum((Fraction(e.duration) for e in evs), Fraction(0))
        for e in evs:
            ev_j[id(e)] = kernel_j[d] * Fraction(e.duration) / span if span > 0 else Fraction(0)
    tasks = {}
    for e in events:
        s0, s1 = Fraction(e.start), Fraction(e.start) + Fraction(e.duration)
        rec = tasks.setdefault(e.task_id, [e.task_name or "", Fraction(0), {}, s0, s1])
        rec[1] += ev_j[id(e)]
        rec[2][e.node] = e.frequency_ghz
        rec[3], rec[4] = min(rec[3], s0), max(rec[4], s1)
    rep = EnergyReport(makespan_s=Fraction(result.makespan))
    rep.per_task = [TaskEnergy(t, r[0], r[4] - r[3], r[1], dict(sorted(r[2].items())))
                    for t, r in sorted(tasks.items())]
    hosted = {}
    for node, d in node_dev.items():
        hosted.setdefault(d, []).append(node)
    for node in sorted(node_dev):
        d = node_dev[node]
        mine = sum((ev_j[id(e)] for e in events if e.node == node), Fraction(0))
        nb = _union_length([(Fraction(e.start), Fraction(e.start) + Fraction(e.duration))
                            for e in events if e.node == node])
        share = idle_j[d] / len(hosted[d])
        rep.per_device.append(DeviceEnergy(node, mine + share, nb, window[d] - nb,
                                           float(nv["devices"][d]["idle_w"])))
    return rep


def kernel_energy_consumption(result, task_id: int) -> float:
    """Measured joules of one submitted task (SYnergy
    ``queue.kernel_energy_consumption(e)``)."""
    for t in measured_energy(result).per_task:
        if t.task_id == task_id:
            return float(t.energy_j)
    raise ValidationError(f"task {task_id} did not execute in this run")


def device_energy_consumption(result, node=None) -> float:
    """Measured joules of one node's device share, or of every device of the
    run when ``node`` is None (SYnergy ``queue.device_energy_consumption()``,
    PAPER.md:129)."""
    nv = (result.measured or {}).get("nvml")
    if not nv:
        raise ValidationError("the run has no NVML readings (use run(..., energy=True))")
    if node is None:
        return float(sum(Fraction(v["energy_j"]) for v in nv["devices"].values()))
    for d in measured_energy(result).per_device:
        if d.node == node:
            return float(d.energy_j)
    raise ValidationError(f"node {node} is not in this run")
