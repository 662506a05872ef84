"""SYnergy on B200: per-kernel energy measured with NVML and frequency
selection over *measured* tables.

The reference picks a frequency per chunk from a modelled device
(energy.py:93-106: exhaustive argmin of E, E*t or E*t^2 over discrete levels,
exact rationals, ties to the higher level).  Here the same selection rule
runs over a table of measured (seconds, joules) per supported SM clock for a
kernel -- ``MeasuredKernel`` -- built by ``sweep``:

* the candidate clocks come from nvmlDeviceGetSupportedGraphicsClocks;
* each point locks the SM clock (nvmlDeviceSetGpuLockedClocks), runs the
  kernel until >= ``seconds`` have elapsed and reads the NVML energy counter
  before/after (the counter updates too coarsely for single launches);
* clock locking changes shared hardware state, so libcq refuses it unless
  CQ_ALLOW_CLOCK_LOCK=1 -- on a pool that forbids tenants from setting clocks
  the sweep reports the running clock only.

``kernel_energy(fn)`` is the paper's ``kernel_energy_consumption(e)``
 as a measurement: joules and seconds of one callable.
"""

import ctypes
import time
from dataclasses import dataclass, field
from fractions import Fraction

from . import _native as N
from .energy import DeviceModel, EnergyTarget
from .errors import NativeError, ValidationError


def supported_sm_clocks(device: int = 0) -> list:
    buf = (ctypes.c_uint * 256)()
    n = ctypes.c_int32(256)
    N.call("cq_nvml_supported_sm_clocks", device, buf, ctypes.byref(n))
    return sorted(set(buf[i] for i in range(n.value)))


def sm_clock(device: int = 0):
    cur, mx = ctypes.c_uint(), ctypes.c_uint()
    N.call("cq_nvml_sm_clock_mhz", device, ctypes.byref(cur), ctypes.byref(mx))
    return cur.value, mx.value


def energy_mj(device: int = 0) -> int:
    v = ctypes.c_uint64()
    N.call("cq_nvml_energy_mj", device, ctypes.byref(v))
    return v.value


def kernel_energy(fn, device: int = 0, seconds: float = 1.0, sync=None):
    """Run ``fn`` repeatedly for >= ``seconds``; returns dict(j_per_call,
    s_per_call, watts, calls, sm_mhz)."""
    e0 = energy_mj(device)
    t0 = time.perf_counter()
    calls = 0
    while True:
        fn()
        calls += 1
        if sync is not None:
            sync()
        if time.perf_counter() - t0 >= seconds and calls >= 3:
            break
    dt = time.perf_counter() - t0
    joules = (energy_mj(device) - e0) / 1000.0
    return {"j_per_call": joules / calls, "s_per_call": dt / calls, "watts": joules / dt,
            "calls": calls, "sm_mhz": sm_clock(device)[0]}


@dataclass
class MeasuredKernel:
    """Measured (seconds, joules) per SM clock (MHz) for one kernel."""

    name: str
    points: dict = field(default_factory=dict)  # mhz -> (seconds, joules)

    def levels(self):
        return sorted(self.points)


def select_measured(kernel: MeasuredKernel, target: EnergyTarget) -> int:
    """Reference selection rule (energy.py:93-106) over measured points:
    MAX_PERF -> the highest clock; else argmin of E, E*t or E*t^2 with exact
    rational comparison and ties to the higher clock."""
    levels = kernel.levels()
    if not levels:
        raise ValidationError(f"kernel '{kernel.name}' has no measured points")
    if target is EnergyTarget.MAX_PERF:
        return levels[-1]
    power = {EnergyTarget.MIN_ENERGY: 0, EnergyTarget.MIN_EDP: 1, EnergyTarget.MIN_ED2P: 2}[target]
    best, best_obj = None, None
    for mhz in levels:
        t, e = (Fraction(x) for x in kernel.points[mhz])
        obj = e * t ** power
        if best_obj is None or obj <= best_obj:
            best, best_obj = mhz, obj
    return best


def sweep(name, fn, device=0, clocks=None, seconds=1.0, sync=None) -> MeasuredKernel:
    """Measure ``fn`` at each clock (locking clocks needs CQ_ALLOW_CLOCK_LOCK=1;
    without it only the running clock is measured)."""
    mk = MeasuredKernel(name)
    if clocks is None:
        clocks = []
    locked = False
    try:
        for mhz in clocks:
            try:
                N.call("cq_nvml_lock_sm_clock", device, mhz)
                locked = True
            except NativeError as exc:
                if exc.status == N.CQ_ERR_PERMISSION:
                    break
                raise
            r = kernel_energy(fn, device, seconds, sync)
            mk.points[mhz] = (r["s_per_call"], r["j_per_call"])
    finally:
        if locked:
            N.call("cq_nvml_reset_sm_clock", device)
    if not mk.points:
        r = kernel_energy(fn, device, seconds, sync)
        mk.points[r["sm_mhz"]] = (r["s_per_call"], r["j_per_call"])
    return mk


def sweep_clocks(supported, fractions=(1.0, 0.75, 0.5)) -> list:
    """The supported SM clocks nearest to the given fractions of the highest
    one (BASELINE: "e.g. max, ~75%, ~50%"), highest first, distinct."""
    if not supported:
        return []
    top = max(supported)
    out = []
    for f in fractions:
        c = min(supported, key=lambda m: (abs(m - f * top), -m))
        if c not in out:
            out.append(c)
    return out


def fit_beta(kernel: MeasuredKernel) -> Fraction:
    """Least-squares beta of the reference time model (energy.py:74-78)
    t(f) = t_ref * (beta + (1 - beta) * f_ref / f) with f_ref the highest
    measured clock and t_ref its time: beta ~ 1 for a memory-bound kernel
    (time independent of the SM clock), ~ 0 for a compute-bound one."""
    levels = kernel.levels()
    if len(levels) < 2:
        raise ValidationError(f"kernel '{kernel.name}': beta needs >= 2 measured clocks")
    f_ref = Fraction(levels[-1])
    t_ref = Fraction(kernel.points[levels[-1]][0])
    # t/t_ref - f_ref/f = beta * (1 - f_ref/f)  ->  one-parameter least squares
    num = den = Fraction(0)
    for mhz in levels[:-1]:
        x = 1 - f_ref / Fraction(mhz)
        y = Fraction(kernel.points[mhz][0]) / t_ref - f_ref / Fraction(mhz)
        num += x * y
        den += x * x
    return num / den


class MeasuredDevice(DeviceModel):
    """A device model backed by measured tables: ``generate_commands`` picks
    a task's clock with ``select_measured`` over its kernel's (seconds,
    joules) points instead of the modelled P(f) and t(f) (reference
    scheduler.py:322-324 calls select_frequency there).  ``kernels`` maps a
    task name (or "*" for every other task) to its ``MeasuredKernel``; tasks
    without a table fall back to the model rule over the measured clocks.
    The levels are the measured clocks in GHz; P(f) for ``account_energy``
    is the mean measured power (J/s) at that clock over the tables."""

    def __init__(self, kernels: dict, p_static_w: float = 0.0, throughput_ref: float = 1e9, node=None):
        clocks = sorted({m for k in kernels.values() for m in k.points})
        if not clocks:
            raise ValidationError("a measured device needs at least one measured clock")
        levels = tuple(Fraction(m, 1000) for m in clocks)
        super().__init__(levels_ghz=tuple(float(x) for x in levels), f_ref_ghz=float(levels[-1]),
                         p_static_w=p_static_w, p_dyn_ref_w=0.0, alpha_exp=3.0,
                         throughput_ref=throughput_ref, node=node)
        object.__setattr__(self, "kernels", dict(kernels))

    def __hash__(self):
        return id(self)

    def __eq__(self, other):
        return self is other

    def table_for(self, task_name: str):
        return self.kernels.get(task_name, self.kernels.get("*"))

    def select_for(self, task_name: str, target: EnergyTarget):
        """GHz for a task under ``target``, or None without a table."""
        table = self.table_for(task_name)
        if table is None:
            return None
        return select_measured(table, target) / 1000.0

    def _power_exact(self, f_ghz: float) -> Fraction:
        mhz = round(float(f_ghz) * 1000)
        watts = [Fraction(k.points[mhz][1]) / Fraction(k.points[mhz][0])
                 for k in self.kernels.values() if mhz in k.points]
        if not watts:
            raise ValidationError(f"no measured power at {f_ghz} GHz")
        return sum(watts, Fraction(0)) / len(watts)


def select_for_task(device, target: EnergyTarget, t_ref, task) -> float:
    """The planner's per-chunk clock: a ``MeasuredDevice`` with a table for
    the task selects over the measurements, any other device uses the
    reference rule (energy.py:93-106) unchanged."""
    from .energy import select_frequency
    if isinstance(device, MeasuredDevice):
        f = device.select_for(task.name, target)
        if f is not None:
            return f
    return select_frequency(device, target, t_ref, task.beta)
