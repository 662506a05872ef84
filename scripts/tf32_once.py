"""One 3xTF32 SGEMM of size m^3 through the executor (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.executor import Placement, Session  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a, b = W.sgemm_inputs(m, m, m)
s = Session(cq.generate_commands(W.sgemm_program(m, m, m, variant="3xtf32", a=a, b=b).graph(), 1),
            Placement(1, 0, (0,)), trace=False)
s.execute()
s.synchronize()
s.close()
print("ok")
