"""Do host->device and device->host copies overlap?  2 GiB each way from
pinned (registered) host arrays, on separate libcq streams."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_06022_b200 import _native as N, executor as E
N.call("cq_init_device", 0)
nb = 2 << 30
src = E.pinned_empty((nb // 4,), np.float32)
dst = E.pinned_empty((nb // 4,), np.float32)
src[:] = 1.0
d1, d2 = ctypes.c_void_p(), ctypes.c_void_p()
N.call("cq_malloc", 0, nb, ctypes.byref(d1))
N.call("cq_malloc", 0, nb, ctypes.byref(d2))
def sync():
    for s in N.ALL_STREAMS:
        N.call("cq_stream_synchronize", 0, s)
def h2d(stream):
    N.call("cq_copy_h2d", 0, stream, d1, ctypes.c_void_p(src.ctypes.data), nb)
def d2h(stream):
    N.call("cq_copy_d2h", 0, stream, ctypes.c_void_p(dst.ctypes.data), d2, nb)
for name, fn in [("h2d alone", lambda: h2d(3)), ("d2h alone", lambda: d2h(4)),
                 ("h2d || d2h (streams 3, 4)", lambda: (h2d(3), d2h(4))),
                 ("h2d || d2h (comm, 4)", lambda: (h2d(2), d2h(4))),
                 ("2x h2d (streams 3, 5) half each", lambda: (
                     N.call("cq_copy_h2d", 0, 3, d1, ctypes.c_void_p(src.ctypes.data), nb // 2),
                     N.call("cq_copy_h2d", 0, 5, ctypes.c_void_p(d1.value + nb // 2), ctypes.c_void_p(src.ctypes.data + nb // 2), nb // 2)))]:
    for rep in range(2):
        sync()
        t0 = time.perf_counter()
        fn()
        sync()
        dt = time.perf_counter() - t0
    print(f"{name}: {dt*1e3:.1f} ms", flush=True)
