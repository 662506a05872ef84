"""3xTF32 CTA-pair SGEMM (MN-major B): tile rasterisation group (CQ_TF32_GROUP_M) and
TMEM accumulation group (CQ_TF32_GROUP_KB, k blocks per drain) at 8192^3 and 16384^3,
interleaved wall-clock timings of whole cq_sgemm calls; C bits compared across settings
only for equal GROUP_KB (the drain grouping changes the fp32 summation order)."""
import ctypes
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
cfgs = [(gm, gkb) for gm, gkb in itertools.product((4, 8, 16, 32), (4, 8))]
for size in (8192, 16384):
    a = torch.rand((size, size), device="cuda") * 2 - 1
    b = torch.rand((size, size), device="cuda") * 2 - 1
    c = torch.empty((size, size), device="cuda")
    torch.cuda.synchronize()
    times = {cfg: [] for cfg in cfgs}
    for rep in range(3):
        for gm, gkb in cfgs:
            os.environ["CQ_TF32_GROUP_M"], os.environ["CQ_TF32_GROUP_KB"] = str(gm), str(gkb)
            N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), size, ctypes.c_void_p(b.data_ptr()), size,
                   ctypes.c_void_p(c.data_ptr()), size, size, size, size)
            N.call("cq_stream_synchronize", 0, 0)
            t0 = time.perf_counter()
            N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), size, ctypes.c_void_p(b.data_ptr()), size,
                   ctypes.c_void_p(c.data_ptr()), size, size, size, size)
            N.call("cq_stream_synchronize", 0, 0)
            times[(gm, gkb)].append(time.perf_counter() - t0)
    for cfg, ts in times.items():
        t = sorted(ts)[len(ts) // 2]
        print(f"{size}^3 group_m={cfg[0]:2d} group_kb={cfg[1]}: {t * 1e3:.2f} ms = {2 * size ** 3 / t / 1e12:.1f} TFLOP/s "
              f"({' '.join(f'{x * 1e3:.2f}' for x in ts)})", flush=True)
