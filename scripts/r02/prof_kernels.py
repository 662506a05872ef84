"""One launch each of the SAXPY (2^28), N-body kick (262,144 bodies) and
3xTF32 SGEMM (8192^3) kernels through the executor, for ncu.

    python scripts/r02/prof_kernels.py saxpy|nbody|sgemm
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402

which = sys.argv[1]
pl = E.Placement(1, 0, (0,))
if which == "saxpy":
    n = 1 << 28
    x, y = W.saxpy_inputs(n, "float32", seed=0)
    prog = W.saxpy_program(n, kind="float32", x=x, y=y)
elif which == "nbody":
    prog = W.nbody_program(262144, steps=1)
else:
    prog = W.sgemm_program(8192, 8192, 8192, variant="3xtf32")
plan = cq.generate_commands(prog.graph(), 1)
s = E.Session(plan, pl, trace=False)
for _ in range(2):
    s.execute(upload=True)
    s.synchronize()
    s.recycle()
s.close()
print("ok", which)
