"""run_batch ms per simulation of the 100-step 16384^2 wave for several
pipeline depths (sessions in flight), beside one simulation's own transfers
copied concurrently (the PCIe floor)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.region import Box  # noqa: E402

H = Wd = 16384
u0, up0 = bench.wave_inputs(H, Wd, (0, H))
plan = cq.generate_commands(W.wave_program(H, Wd, steps=100, kind="float32", c=0.25, u0=u0, up0=up0).graph(), 1)
box = Box((0, 0), (H, Wd))
outs = [{"u": E.pinned_empty((H, Wd), np.float32, box), "up": E.pinned_empty((H, Wd), np.float32, box)}
        for _ in range(6)]
E.run_batch(plan, [(None, outs[k % 3]) for k in range(6)], gather="root", depth=3)
for rep in range(2):
    for depth in (1, 2, 3, 4):
        t0 = time.perf_counter()
        E.run_batch(plan, [(None, outs[k % depth]) for k in range(12)], gather="root", depth=depth)
        print(f"depth {depth}: {(time.perf_counter() - t0) / 12 * 1e3:.1f} ms/simulation", flush=True)
print("floor", bench.pcie_floor(0, pattern=(1 << 30, 2 << 30))["pattern_ms"], "ms", flush=True)
