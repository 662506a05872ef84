"""A/B timing of the 3xTF32 kernel variants in one process (env read per call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import workloads as W
from paper_2505_06022_b200.executor import Session, Placement
from oracle import native as onat

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a, b = W.sgemm_inputs(m, m, m)
prog = W.sgemm_program(m, m, m, variant="3xtf32", a=a, b=b)
s = Session(cq.generate_commands(prog.graph(), 1), Placement(1, 0, (0,)))
s.execute(); s.synchronize(); s.recycle()
modes = {"2sm_g8": {"CQ_TF32_2SM": "1", "CQ_TF32_GROUP_M": "8"},
         "2sm_g16": {"CQ_TF32_2SM": "1", "CQ_TF32_GROUP_M": "16"},
         "2sm_g4": {"CQ_TF32_2SM": "1", "CQ_TF32_GROUP_M": "4"},
         "1sm": {"CQ_TF32_2SM": "0"}}
ref_rows = np.arange(0, m, m // 64)
c, cabs = onat.sgemm_rows(a, b, ref_rows)
for rnd in range(2):
    for name, env in modes.items():
        os.environ.update(env)
        s.execute(upload=False); s.synchronize(); s.recycle()
        m0 = s.mark()
        for _ in range(4):
            s.execute(upload=False)
        m1 = s.mark(); s.synchronize()
        ms = s.elapsed_ms(m0[0], m1[0]) / 4
        s.recycle()
        err = (np.abs(s.results()["C"][ref_rows] - c) / cabs).max() if rnd == 0 else float("nan")
        print(f"round {rnd} {name}: {ms:.2f} ms {2*m**3/ms/1e9:.1f} TFLOP/s err {err:.3e}", flush=True)
s.close()
