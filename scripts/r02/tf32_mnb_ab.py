"""3xTF32 SGEMM 8192^3 and 16384^3: B read MN-major from [k, n] (CQ_TF32_MNB=1,
default) vs the transposed Bt_hi / Bt_lo copies, interleaved wall-clock
timings of whole cq_sgemm calls (split pass + GEMM) on libcq's stream."""
import ctypes
import os
import sys
import time

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

    def call():
        N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), size, ctypes.c_void_p(b.data_ptr()), size,
               ctypes.c_void_p(c.data_ptr()), size, size, size, size)

    for rep in range(5):
        for mnb in ("1", "0"):
            os.environ["CQ_TF32_MNB"] = mnb
            call()   # warm (scratch)
            N.call("cq_stream_synchronize", 0, 0)
            t0 = time.perf_counter()
            call()
            N.call("cq_stream_synchronize", 0, 0)
            times[mnb].append(time.perf_counter() - t0)
    for mnb, ts in times.items():
        t = sorted(ts)[len(ts) // 2]
        print(f"{size}^3 mnb={mnb}: {t * 1e3:.2f} ms = {2 * size ** 3 / t / 1e12:.1f} TFLOP/s "
              f"(all: {' '.join(f'{x * 1e3:.2f}' for x in ts)})", flush=True)
