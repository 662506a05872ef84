"""e2e leg of bench.py in isolation, with the process optionally bound to
the CPUs local to the GPU (argv[1] == "bind"): run_batch ms per simulation
over three timed batches, the sequential run() beside it, and where the
host buffers' pages live (/proc/self/numa_maps)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
BIND = len(sys.argv) > 1 and sys.argv[1] == "bind"


def local_cpus(dev=0):
    import subprocess
    bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                         capture_output=True, text=True).stdout.strip().lower()
    bus = bus[4:] if len(bus.split(":")[0]) == 8 else bus
    path = f"/sys/bus/pci/devices/{bus}"
    try:
        cpus = open(path + "/local_cpulist").read().strip()
        node = open(path + "/numa_node").read().strip()
    except OSError as exc:
        return None, None, str(exc)
    out = set()
    for part in cpus.split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out, node, cpus


cpus, node, txt = local_cpus()
print(f"GPU0 numa_node={node} local_cpulist={txt}; process affinity {len(os.sched_getaffinity(0))} cpus", flush=True)
if BIND and cpus:
    os.sched_setaffinity(0, cpus)
    print(f"bound to {len(cpus)} cpus", flush=True)

import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.region import Box  # noqa: E402

H = Wd = 16384
u0, up0 = bench.wave_inputs(H, Wd, (0, H))
prog = W.wave_program(H, Wd, steps=100, kind="float32", c=0.25, u0=u0, up0=up0)
plan = cq.generate_commands(prog.graph(), 1)
box = Box((0, 0), (H, Wd))
outs = [{"u": E.pinned_empty((H, Wd), np.float32, box), "up": E.pinned_empty((H, Wd), np.float32, box)}
        for _ in range(3)]


def numa_of(arr):
    start = arr.__array_interface__["data"][0]
    for line in open("/proc/self/numa_maps"):
        addr = int(line.split()[0], 16)
        if addr <= start < addr + arr.nbytes + (1 << 22) and addr + 4096 > start - (1 << 21):
            return " ".join(x for x in line.split() if x.startswith("N"))
    return "?"


print("pages: u0", numa_of(u0), "| outs", [numa_of(o["u"]) for o in outs], flush=True)
E.run_batch(plan, [(None, outs[k % 3]) for k in range(6)], gather="root", depth=3)
for rep in range(3):
    t0 = time.perf_counter()
    E.run_batch(plan, [(None, outs[k % 3]) for k in range(10)], gather="root", depth=3)
    print(f"run_batch 10 jobs: {(time.perf_counter() - t0) * 100:.1f} ms/job", flush=True)
t0 = time.perf_counter()
for _ in range(3):
    E.run(plan, gather="root", out=outs[0], trace=False)
print(f"run(): {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms/sim", flush=True)
print("link", bench.pcie_floor(0, pattern=(1 << 30, 2 << 30)), flush=True)
