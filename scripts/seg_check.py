"""Interleaved, repeated timing of the fused wave pass: the automatic
rows-per-block choice against fixed segments (CQ_FUSED_SEG, read per
launch), KL = 8 and 4, several slab heights.  A throw-away round first, so
freshly allocated memory does not bias the first column."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
w = 16384
for h in (16384, 8192, 4096, 2048, 1024, 512):
    t = [torch.rand((h, w), device="cuda") for _ in range(4)]
    torch.cuda.synchronize()

    def view(x):
        v = N.CqView()
        v.ptr = x.data_ptr()
        v.alloc = N.box3((0, 0), (h, w))
        v.stride[:] = [h * w, w, 1]
        return v
    vs = [view(x) for x in t]
    ext = N.box3((0, 0), (h, w))
    for kl, fixed in ((8, (224, 128, 64)), (4, (128, 64, 32))):
        for rep in range(3):
            row = []
            for seg in ("auto",) + fixed:
                if seg == "auto":
                    os.environ.pop("CQ_FUSED_SEG", None)
                else:
                    os.environ["CQ_FUSED_SEG"] = str(seg)

                def go(n):
                    for _ in range(n):
                        N.call("cq_wave5_fused", 0, 0, N.CQ_F32, kl, ctypes.byref(vs[0]), ctypes.byref(vs[1]),
                               ctypes.byref(vs[2]), ctypes.byref(vs[3]), 0, h, 0, h, ctypes.byref(ext),
                               0.25, 2.0, 4.0)
                    N.call("cq_stream_synchronize", 0, 0)
                go(3)
                reps = max(10, int(3e4 // h))
                t0 = time.perf_counter()
                go(reps)
                row.append(f"{seg}:{(time.perf_counter() - t0) / reps * 1e3:.3f}")
            if rep:
                print(f"h={h:6d} KL={kl} ms/pass " + " ".join(row), flush=True)
    del t, vs
os.environ.pop("CQ_FUSED_SEG", None)
