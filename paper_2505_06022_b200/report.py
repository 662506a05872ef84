"""report.json / trace.json / buf_<name>.json from a measured B200 run.

Same schema and key order as the reference CLI (pkg/src/clusterq/cli.py:85-151,
docs/formats.md:130-186), filled from the executor's measured trace (CUDA
event times) instead of logical time.  The model energy is the reference's
``account_energy`` over those durations; when the run measured NVML energy
(``run(..., energy=True)``) a ``measured`` section carries the NVML joules
per device and per task (``measure.measured_energy``) --
kernel_energy_consumption / device_energy_consumption of the paper's SYnergy
API as real readings.
"""

import json
import os

from .energy import account_energy
from .executor import trace_to_chrome


def build_report(result, devices=None) -> dict:
    """Reference report.json dict for a ``RunResult``."""
    devices = devices if devices is not None else result.plan.devices
    energy = account_energy(result.trace, devices, result.makespan)
    pushes = [ev for ev in result.trace if ev.kind == "push"]
    out = {
        "makespan_s": float(energy.makespan_s),
        "per_task": [
            {"id": t.task_id, "name": t.name, "duration_s": float(t.duration_s),
             "energy_j": float(t.energy_j),
             "frequency_ghz_per_node": {str(n): f for n, f in t.frequency_ghz_per_node.items()}}
            for t in energy.per_task
        ],
        "per_device": [
            {"node": d.node, "energy_j": float(d.energy_j), "busy_s": float(d.busy_s),
             "idle_s": float(d.idle_s)}
            for d in energy.per_device
        ],
        "transfers": {"count": len(pushes), "total_bytes": sum(ev.bytes for ev in pushes)},
    }
    if result.measured:
        out["measured"] = {k: v for k, v in result.measured.items() if k != "nvml"}
        if "nvml" in result.measured:
            from .measure import measured_energy
            m = measured_energy(result)
            out["measured"]["per_task"] = [{"id": t.task_id, "name": t.name, "energy_j": float(t.energy_j)}
                                           for t in m.per_task]
            out["measured"]["per_device"] = [{"node": d.node, "energy_j": float(d.energy_j),
                                              "busy_s": float(d.busy_s), "idle_s": float(d.idle_s),
                                              "idle_w": d.static_power_w} for d in m.per_device]
    return out


def trace_document(result) -> dict:
    return {"traceEvents": trace_to_chrome(result.trace)}


def buffer_dump(name, arr, buffer) -> dict:
    flat = arr.reshape(-1)
    if buffer.element_kind == "int64":
        values = [int(v) for v in flat]
    else:
        values = [float(v) for v in flat]
    return {"name": name, "extent": list(buffer.extent.shape), "element_kind": buffer.element_kind,
            "values": values}


def write_outputs(result, outdir, devices=None, dump_buffers=True):
    """Write report.json, trace.json and buf_<name>.json like `clusterq run`."""
    os.makedirs(outdir, exist_ok=True)

    def dump(path, obj):
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(obj, fh, indent=2)
            fh.write("\n")

    dump(os.path.join(outdir, "report.json"), build_report(result, devices))
    dump(os.path.join(outdir, "trace.json"), trace_document(result))
    if dump_buffers:
        buffers = result.plan.graph.buffers
        for name, arr in result.buffers.items():
            dump(os.path.join(outdir, f"buf_{name}.json"), buffer_dump(name, arr, buffers[name]))
