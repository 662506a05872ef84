"""Why bench.py's e2e (run_batch, 3 in flight) sometimes runs slower than one
run at a time: the same e2e leg timed fresh, after a device-resident session
(graph capture + energy loop, as bench.py does before it), with several job
counts, and per-job host timelines."""
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
pl = E.Placement(1, 0, (0,))
u0, up0 = bench.wave_inputs(H, Wd, (0, H))
prog = W.wave_program(H, Wd, steps=100, kind="float32", c=0.25, u0=u0, up0=up0)
plan = cq.generate_commands(prog.graph(), 1)
box = Box((0, 0), (H, Wd))
outs = [{"u": E.pinned_empty((H, Wd), np.float32, box), "up": E.pinned_empty((H, Wd), np.float32, box)}
        for _ in range(3)]


def e2e(tag, jobs=5, depth=3):
    E.run_batch(plan, [(None, outs[k % depth]) for k in range(depth)], depth=depth)
    t0 = time.perf_counter()
    E.run_batch(plan, [(None, outs[k % depth]) for k in range(jobs)], depth=depth)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    E.run(plan, out=outs[0], trace=False)
    sync = time.perf_counter() - t1
    print(f"{tag}: run_batch {jobs} jobs depth {depth}: {dt / jobs * 1e3:.1f} ms/job; one run {sync * 1e3:.1f} ms",
          flush=True)


e2e("fresh")
e2e("fresh, 10 jobs", jobs=10)
# what bench.py does before its e2e leg: a session, graph replays, an energy loop
sess = E.Session(plan, pl, trace=True)
sess.execute(upload=True)
sess.synchronize()
sess.recycle()
sess.capture()
for _ in range(150):
    sess.replay(1)
sess.synchronize()
sess.close()
e2e("after device-resident replays")
e2e("after device-resident replays, 10 jobs", jobs=10)
e2e("depth 2", depth=2)
print("pcie", bench.pcie_floor(0), flush=True)
e2e("after pcie_floor")
