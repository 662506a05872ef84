"""Host timeline of bench.py's e2e leg in a fresh process (the slow case of
e2e_diag.py: the first timed run_batch after one warm-up batch)."""
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
t_start = time.perf_counter()
u0, up0 = bench.wave_inputs(H, Wd, (0, H))
print(f"inputs {time.perf_counter() - t_start:.2f} s", flush=True)
prog = W.wave_program(H, Wd, steps=100, kind="float32", c=0.25, u0=u0, up0=up0)
plan = cq.generate_commands(prog.graph(), 1)
box = Box((0, 0), (H, Wd))
t = time.perf_counter()
outs = [{"u": E.pinned_empty((H, Wd), np.float32, box), "up": E.pinned_empty((H, Wd), np.float32, box)}
        for _ in range(3)]
print(f"outs pinned {time.perf_counter() - t:.2f} s", flush=True)
log = []
for name in ("execute", "issue_results", "finish_results", "__init__", "close"):
    orig = getattr(E.Session, name)

    def wrap(self, *a, _o=orig, _n=name, **k):
        t = time.perf_counter()
        r = _o(self, *a, **k)
        log.append((_n, id(self) % 1000, t, time.perf_counter()))
        return r
    setattr(E.Session, name, wrap)
for label, jobs in (("warm", 3), ("timed", 5), ("again", 5), ("again", 5)):
    log.clear()
    t0 = time.perf_counter()
    E.run_batch(plan, [(None, outs[k % 3]) for k in range(jobs)], depth=3)
    total = time.perf_counter() - t0
    print(f"{label} {jobs} jobs: {total * 1e3:.1f} ms ({total / jobs * 1e3:.1f} ms/job)", flush=True)
    for n, sid, a, b in log:
        if b - a > 0.002:
            print(f"   {n:15s} s{sid:03d} {1e3 * (a - t0):8.1f} -> {1e3 * (b - t0):8.1f} ms ({1e3 * (b - a):7.1f})",
                  flush=True)
