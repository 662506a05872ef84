"""3xTF32 SGEMM 8192^3 and 16384^3: interleaved wall-clock timings of whole
cq_sgemm calls under two values of one environment knob.

    python scripts/r02/tf32_env_ab.py CQ_TF32_INSPLIT 1 0
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2505_06022_b200 import _native as N  # noqa: E402

name, vals = sys.argv[1], sys.argv[2:]
N.call("cq_init_device", 0)
for size in (8192, 16384):
    a = torch.rand((size, size), device="cuda") * 2 - 1
    b = torch.rand((size, size), device="cuda") * 2 - 1
    c = torch.empty((size, size), device="cuda")
    torch.cuda.synchronize()
    times = {v: [] for v in vals}

    def call():
        N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), size, ctypes.c_void_p(b.data_ptr()), size,
               ctypes.c_void_p(c.data_ptr()), size, size, size, size)

    for rep in range(6):
        for v in (vals if rep % 2 == 0 else vals[::-1]):
            os.environ[name] = v
            call()
            N.call("cq_stream_synchronize", 0, 0)
            time.sleep(0.2)   # let the power state settle between arms
            t0 = time.perf_counter()
            call()
            N.call("cq_stream_synchronize", 0, 0)
            times[v].append(time.perf_counter() - t0)
    for v, ts in times.items():
        t = sorted(ts)[len(ts) // 2]
        print(f"{size}^3 {name}={v}: median {t * 1e3:.2f} ms = {2 * size ** 3 / t / 1e12:.1f} TFLOP/s "
              f"(all: {' '.join(f'{x * 1e3:.2f}' for x in ts)})", flush=True)
