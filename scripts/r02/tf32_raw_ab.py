"""3xTF32 SGEMM 16384^3 (and 8192^3): A as its own hi part (CQ_TF32_RAW_HI=1,
default) vs the masked copy, interleaved CUDA-event timings."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
for size in (8192, 16384):
    a = torch.rand((size, size), device="cuda") * 2 - 1
    b = torch.rand((size, size), device="cuda") * 2 - 1
    c = torch.empty((size, size), device="cuda")
    torch.cuda.synchronize()
    times = {"1": [], "0": []}
    for rep in range(4):
        for raw in ("1", "0"):
            os.environ["CQ_TF32_RAW_HI"] = raw
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), size, ctypes.c_void_p(b.data_ptr()), size,
                   ctypes.c_void_p(c.data_ptr()), size, size, size, size)   # warm (scratch) on libcq's stream
            N.call("cq_stream_synchronize", 0, 0)
            s = torch.cuda.current_stream()
            e0.record(s)
            torch.cuda.synchronize()
            import time
            t0 = time.perf_counter()
            N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), size, ctypes.c_void_p(b.data_ptr()), size,
                   ctypes.c_void_p(c.data_ptr()), size, size, size, size)
            N.call("cq_stream_synchronize", 0, 0)
            times[raw].append(time.perf_counter() - t0)
    for raw, ts in times.items():
        t = sorted(ts)[len(ts) // 2]
        print(f"{size}^3 raw_hi={raw}: {t * 1e3:.2f} ms = {2 * size ** 3 / t / 1e12:.1f} TFLOP/s", flush=True)
