"""Sweep of the fused wave pass's rows-per-block (CQ_FUSED_SEG, read per
launch) at several slab heights, KL = 8 and 4; 'auto' is the default
choice.  Wall clock over many queued launches, one synchronize."""
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
    for kl in (8, 4):
        row = []
        for seg in ("auto", 32, 48, 64, 96, 128, 160, 192, 224, 256):
            if seg == "auto":
                os.environ.pop("CQ_FUSED_SEG", None)
            else:
                os.environ["CQ_FUSED_SEG"] = str(seg)

            def go(n):
                for _ in range(n):
                    N.call("cq_wave5_fused", 0, 0, N.CQ_F32, kl, ctypes.byref(vs[0]), ctypes.byref(vs[1]),
                           ctypes.byref(vs[2]), ctypes.byref(vs[3]), 0, h, 0, h, ctypes.byref(ext), 0.25, 2.0, 4.0)
                N.call("cq_stream_synchronize", 0, 0)
            go(3)
            reps = max(10, int(3e4 // h))
            t0 = time.perf_counter()
            go(reps)
            dt = (time.perf_counter() - t0) / reps
            row.append(f"{seg}:{dt * 1e3:.3f}")
        print(f"h={h:6d} KL={kl} ms/pass " + " ".join(row), flush=True)
    del t, vs
os.environ.pop("CQ_FUSED_SEG", None)
