"""GPU check of the 3xTF32 tcgen05 SGEMM against the CPU oracle, then timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import workloads as W
from paper_2505_06022_b200.executor import run, Session, Placement
from oracle import native as onat

pl = Placement(1, 0, (0,))
for (m, n, k) in [(128, 128, 32), (256, 256, 256), (384, 512, 1024), (1000, 777, 520), (2048, 2048, 2048)]:
    a, b = W.sgemm_inputs(m, n, k)
    for variant in ("3xtf32", "ffma"):
        prog = W.sgemm_program(m, n, k, variant=variant, a=a, b=b)
        res = run(cq.generate_commands(prog.graph(), 1), placement=pl)
        rows = np.arange(0, m, max(1, m // 64))
        c, cabs = onat.sgemm_rows(a, b, rows)
        err = np.abs(res.buffers["C"][rows] - c) / cabs
        print(f"{variant} {m}x{n}x{k}: max normalised err {err.max():.3e}", flush=True)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a, b = W.sgemm_inputs(m, m, m)
for variant in ("3xtf32", "ffma"):
    prog = W.sgemm_program(m, m, m, variant=variant, a=a, b=b)
    s = Session(cq.generate_commands(prog.graph(), 1), pl)
    s.execute(); s.synchronize(); s.recycle()
    m0 = s.mark()
    for _ in range(3):
        s.execute(upload=False)
    m1 = s.mark(); s.synchronize()
    ms = s.elapsed_ms(m0[0], m1[0]) / 3
    print(f"{variant} {m}^3: {ms:.2f} ms  {2*m**3/ms/1e9:.1f} TFLOP/s", flush=True)
    if variant == "3xtf32":
        out = s.results()
        rows = np.arange(0, m, m // 64)
        c, cabs = onat.sgemm_rows(a, b, rows)
        print("  err", (np.abs(out["C"][rows] - c) / cabs).max(), flush=True)
    s.close()
