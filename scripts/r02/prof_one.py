"""One bounded (FMA-form) KL pass at 16384^2 under the current CQ_FUSED_*
environment, for ncu.   python scripts/r02/prof_one.py KL"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
kl = int(sys.argv[1]) if len(sys.argv) > 1 else 8
h = w = 16384
t = [torch.rand((h, w), device="cuda") for _ in range(4)]
bound = torch.tensor([1.0, 0.0], device="cuda", dtype=torch.float32)
torch.cuda.synchronize()


def view(x):
    v = N.CqView()
    v.ptr = x.data_ptr()
    v.alloc = N.box3((0, 0), (h, w))
    v.stride[:] = [h * w, w, 1]
    return v


vs = [view(x) for x in t]
ext = N.box3((0, 0), (h, w))
for i in range(3):
    N.call("cq_wave5_fused_bounded", 0, 0, N.CQ_F32, kl, ctypes.byref(vs[0]), ctypes.byref(vs[1]),
           ctypes.byref(vs[2]), ctypes.byref(vs[3]), 0, h, 0, h, ctypes.byref(ext), 0.25, 2.0, 4.0,
           ctypes.c_void_p(bound.data_ptr()), ctypes.c_void_p(bound.data_ptr() + 4))
N.call("cq_stream_synchronize", 0, 0)
print("ok", kl, float(bound[1]))
