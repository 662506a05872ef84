"""report.json / trace.json (the reference CLI's outputs, cli.py:85-151) from a
measured B200 run: a 16384 x 16384 fp32 wave, 800 steps, 4 plan nodes on one GPU
(temporally blocked passes, lanes), NVML energy measured around the run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.executor import Placement, run  # noqa: E402
from paper_2505_06022_b200.report import write_outputs  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/report_demo"
prog = W.wave_program(16384, 16384, steps=800, kind="float32")
plan = cq.generate_commands(prog.graph(), 4)
res = run(plan, placement=Placement(1, 0, (0,)), energy=True)
write_outputs(res, out, dump_buffers=False)
print("wrote", sorted(os.listdir(out)), "makespan", float(res.makespan), "measured", res.measured)
