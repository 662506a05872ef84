"""N-body kick: r^-3 via rsqrt*rcp on a fixed subset of j slots (CQ_NBODY_RCP
mask over each 8 slots) vs rsqrt^3 everywhere -- interleaved timing of one
262,144-body kick and the accuracy against the float64 oracle."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_06022_b200 import _native as N  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from oracle import native as onat  # noqa: E402

N.call("cq_init_device", 0)
n, eps2, dt = 262144, 1e-2, 1e-3
pos, vel = W.nbody_inputs(n)
P = torch.from_numpy(pos).cuda()
V = torch.from_numpy(vel).cuda()
out = torch.empty_like(V)
torch.cuda.synchronize()
idx = np.random.default_rng(0).choice(n, 1024, replace=False)
want = onat.nbody_accel_idx(pos, idx, eps2)


class Ev:
    def __init__(self):
        h = ctypes.c_uint64()
        N.call("cq_event_create", 0, 1, ctypes.byref(h))
        self.h = h.value

    def record(self):
        N.call("cq_event_record", ctypes.c_uint64(self.h), 0, 0)

    def ms(self, o):
        v = ctypes.c_float()
        N.call("cq_event_elapsed_ms", ctypes.c_uint64(self.h), ctypes.c_uint64(o.h), ctypes.byref(v))
        return v.value


def kick():
    N.call("cq_nbody_kick", 0, 0, ctypes.c_void_p(P.data_ptr()), n, ctypes.c_void_p(V.data_ptr()),
           ctypes.c_void_p(out.data_ptr()), 0, n, ctypes.c_float(eps2), ctypes.c_float(dt))


masks = ["0", "0x11", "0x15", "0x55"]
times = {m: [] for m in masks}
e0, e1 = Ev(), Ev()
for rep in range(5):
    for m in masks:
        os.environ["CQ_NBODY_RCP"] = m
        kick()
        e0.record()
        kick()
        kick()
        e1.record()
        N.call("cq_stream_synchronize", 0, 0)
        times[m].append(e0.ms(e1) / 2)
for m in masks:
    os.environ["CQ_NBODY_RCP"] = m
    kick()
    N.call("cq_stream_synchronize", 0, 0)
    got = out.cpu().numpy()[idx, :3].astype(np.float64) / dt
    err = (np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)).max()
    t = sorted(times[m])[len(times[m]) // 2]
    print(f"mask {m}: {t:.3f} ms median = {20 * n * n / t / 1e9:.0f} GFLOP/s; max rel err {err:.2e}", flush=True)
