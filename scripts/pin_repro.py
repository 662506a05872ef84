"""Reproduce rank-0 host uploads of a 2-rank weak-scaled wave bench on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.region import Box  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
size = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
if "--torch" in sys.argv:
    import torch  # noqa: F401
H, Wd = size * world, size
rows = (0, size + 1)
box = Box((rows[0], 0), (rows[1], Wd))
u0 = E.pinned_empty((H, Wd), np.float32, box)
u0[rows[0]:rows[1]] = 1.0
up0 = E.pinned_empty((H, Wd), np.float32, box)
up0[rows[0]:rows[1]] = 1.0
print("pinned spans", [(hex(s), e - s) for s, e in E._pinned], flush=True)
print("u0 base", hex(u0.ctypes.data), "up0 base", hex(up0.ctypes.data), flush=True)
prog = W.wave_program(H, Wd, steps=2, kind="float32", u0=u0, up0=up0)
plan = cq.generate_commands(prog.graph(), world)
sess = E.Session(plan, E.Placement(world, 0, (0,)), trace=False)
try:
    t0 = time.perf_counter()
    sess.seed_node0()
    sess.synchronize()
    print("seed ok", time.perf_counter() - t0, flush=True)
except Exception as exc:  # noqa: BLE001
    print("seed FAILED:", exc, flush=True)
    print("pinned spans after", [(hex(s), e - s) for s, e in E._pinned], flush=True)
