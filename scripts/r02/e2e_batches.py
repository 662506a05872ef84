"""bench.py's e2e leg repeated: 8 timed run_batch calls of 5 simulations,
with the time each job's read-back completes (host clock), to see what an
occasional 3x slower batch consists of."""
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
        for _ in range(3)]
marks = []
orig = E.Session.finish_results


def finish(self, state):
    r = orig(self, state)
    marks.append(time.perf_counter())
    return r


E.Session.finish_results = finish
closes = []
orig_close = E.Session.close


slow_calls = []
orig_call = E.N.call


def timed_call(name, *args):
    a = time.perf_counter()
    r = orig_call(name, *args)
    dt = time.perf_counter() - a
    if dt > 0.005:
        slow_calls.append((name, round(dt * 1e3)))
    return r


def close(self):
    a = time.perf_counter()
    E.N.call = timed_call
    try:
        orig_close(self)
    finally:
        E.N.call = orig_call
    closes.append(time.perf_counter() - a)


E.Session.close = close
import gc  # noqa: E402
if len(sys.argv) > 1 and sys.argv[1] == "nogc":
    gc.disable()
    print("gc disabled", flush=True)
gc.callbacks.append(lambda phase, info: print(f"   gc {phase} gen{info['generation']} at {time.perf_counter():.3f}",
                                             flush=True) if phase == "start" and info["generation"] == 2 else None)
E.run_batch(plan, [(None, outs[k % 3]) for k in range(6)], gather="root", depth=3)
for rep in range(8):
    marks.clear()
    closes.clear()
    slow_calls.clear()
    t0 = time.perf_counter()
    E.run_batch(plan, [(None, outs[k % 3]) for k in range(5)], gather="root", depth=3)
    t1 = time.perf_counter()
    print(f"batch {rep}: {(t1 - t0) * 200:.1f} ms/sim; read-backs done at " +
          " ".join(f"{(m - t0) * 1e3:.0f}" for m in marks) + " ms; closes " +
          " ".join(f"{c * 1e3:.0f}" for c in closes) + f" ms (t={t1:.3f}) slow calls {slow_calls}", flush=True)
