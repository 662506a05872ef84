import ctypes, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2505_06022_b200 import _native as N
N.call("cq_init_device", 0)
h = w = 16384
t = [torch.rand((h, w), device="cuda") for _ in range(4)]
bound = torch.tensor([1.0, 0.0], device="cuda")
torch.cuda.synchronize()
def view(x):
    v = N.CqView(); v.ptr = x.data_ptr(); v.alloc = N.box3((0, 0), (h, w)); v.stride[:] = [h * w, w, 1]; return v
vs = [view(x) for x in t]
ext = N.box3((0, 0), (h, w))
for rep in range(3):
    row = []
    for seg in (224, 208, 181, 161, 224, 208):
        os.environ["CQ_FUSED_SEG"] = str(seg)
        def go(n):
            for _ in range(n):
                N.call("cq_wave5_fused_bounded", 0, 0, N.CQ_F32, 8, ctypes.byref(vs[0]), ctypes.byref(vs[1]), ctypes.byref(vs[2]), ctypes.byref(vs[3]), 0, h, 0, h, ctypes.byref(ext), 0.25, 2.0, 4.0, ctypes.c_void_p(bound.data_ptr()), ctypes.c_void_p(bound.data_ptr() + 4))
            N.call("cq_stream_synchronize", 0, 0)
        go(3); t0 = time.perf_counter(); go(20); row.append(f"{seg}:{(time.perf_counter()-t0)/20*1e3:.3f}")
    print("KL8 fast 16384^2 ms/pass", " ".join(row), flush=True)
