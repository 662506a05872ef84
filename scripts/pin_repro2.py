"""Repro: rank-0 view of a 2-rank fused wave run materialises rows [0, 16392)
of a host array pinned only over rows [0, 16385)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import executor as E, workloads as W
from paper_2505_06022_b200.region import Box
H, Wd = 32768, 16384
box = Box((0, 0), (16385, Wd))
u0 = E.pinned_empty((H, Wd), np.float32, box)
up0 = E.pinned_empty((H, Wd), np.float32, box)
u0[:16385] = 1.0
up0[:16385] = 1.0
print("pinned spans:", [(hex(s), hex(e)) for s, e in E._pinned], flush=True)
prog = W.wave_program(H, Wd, steps=12, kind="float32", u0=u0, up0=up0)
plan = cq.generate_commands(prog.graph(), 2)
s = E.Session(plan, E.Placement(2, 0, (0,)))
print("chains:", [(c.depth, c.rows) for c in s.chains], flush=True)
for (n, b), v in s.views.items():
    print("view", n, b, v.box, flush=True)
    arr = s.host_array(b)
    print("  base", hex(arr.ctypes.data), "span", [hex(x) for x in E._byte_span(arr, v.box)],
          "state", E._pin_state(*E._byte_span(arr, v.box)), flush=True)
print("pinned spans after session:", [(hex(s_), hex(e)) for s_, e in E._pinned], flush=True)
s.seed_node0()
s.synchronize()
print("seed ok", flush=True)
