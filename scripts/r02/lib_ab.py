"""Time the bounded (FMA-form) KL=8 and KL=4 fused passes at 16384^2 with the
libcq named by CQ_LIB, and check them bit-exact against KL one-step launches
(the exact DSL form) on a 4096^2 grid and a row slab.  Run once per library
variant, alternating, on one box:  CQ_LIB=... python scripts/r02/lib_ab.py"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402  (device memory only)

from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
K2, K4, C = 2.0, 4.0, 0.25
bound = torch.zeros(2, device="cuda", dtype=torch.float32)


def view(t, h, w):
    v = N.CqView()
    v.ptr = t.data_ptr()
    v.alloc = N.box3((0, 0), (h, w))
    v.stride[:] = [h * w, w, 1]
    return v


def fused(vs, h, w, kl, rows=None, fast=True):
    ext = N.box3((0, 0), (h, w))
    lo, hi = rows or (0, h)
    bound[0] = 1.0 if fast else float("inf")
    N.call("cq_wave5_fused_bounded", 0, 0, N.CQ_F32, kl, ctypes.byref(vs[0]), ctypes.byref(vs[1]),
           ctypes.byref(vs[2]), ctypes.byref(vs[3]), lo, hi, lo + (kl if rows else 0), hi - (kl if rows else 0),
           ctypes.byref(ext), C, K2, K4, ctypes.c_void_p(bound.data_ptr()), ctypes.c_void_p(bound.data_ptr() + 4))


def check(h, w, kl, slab, fast):
    g = torch.Generator(device="cuda").manual_seed(5)
    a, b = torch.rand((h, w), device="cuda", generator=g), torch.rand((h, w), device="cuda", generator=g)
    a[:, :5] *= 1e-37
    ol, op = torch.full_like(a, float("nan")), torch.full_like(a, float("nan"))
    torch.cuda.synchronize()
    rows = (h // 4, 3 * h // 4) if slab else None
    fused([view(x, h, w) for x in (a, b, ol, op)], h, w, kl, rows, fast)
    x, y = a.clone(), b.clone()
    torch.cuda.synchronize()
    ext = N.box3((0, 0), (h, w))
    for _ in range(kl):
        N.call("cq_wave5", 0, 0, N.CQ_F32, ctypes.byref(view(x, h, w)), ctypes.byref(view(y, h, w)),
               ctypes.byref(view(y, h, w)), ctypes.byref(ext), ctypes.byref(ext), C, K2, K4)
        x, y = y, x
    N.call("cq_stream_synchronize", 0, 0)
    s = slice(h // 4 + kl, 3 * h // 4 - kl) if slab else slice(0, h)
    return torch.equal(ol[s].view(torch.int32), x[s].view(torch.int32)) and \
        torch.equal(op[s].view(torch.int32), y[s].view(torch.int32))


SHAPES = ((4096, 4096), (517, 384), (1000, 1000), (40, 1024), (300, 2176), (2048, 16384), (129, 256))
ok = True
for (h, w) in SHAPES:
    for kl in (4, 8):
        for slab in (False, True):
            for fast in (False, True):
                if not check(h, w, kl, slab, fast):
                    ok = False
                    print(f"MISMATCH {h}x{w} KL={kl} slab={slab} fast={fast}", flush=True)


class Ev:
    def __init__(self):
        h = ctypes.c_uint64()
        N.call("cq_event_create", 0, 1, ctypes.byref(h))
        self.h = h.value

    def record(self):
        N.call("cq_event_record", ctypes.c_uint64(self.h), 0, 0)

    def ms(self, other):
        v = ctypes.c_float()
        N.call("cq_event_elapsed_ms", ctypes.c_uint64(self.h), ctypes.c_uint64(other.h), ctypes.byref(v))
        return v.value


h = w = 16384
t = [torch.rand((h, w), device="cuda") for _ in range(4)]
vs = [view(x, h, w) for x in t]
torch.cuda.synchronize()
res = {}
for kl in (8, 4, 8):
    evs = [Ev() for _ in range(24)]
    for i in range(3 + 12):
        order = vs if i % 2 == 0 else vs[2:] + vs[:2]   # ping-pong between the two pairs
        if i >= 3:
            evs[2 * (i - 3)].record()
        fused(order, h, w, kl)
        if i >= 3:
            evs[2 * (i - 3) + 1].record()
    N.call("cq_stream_synchronize", 0, 0)
    ts = sorted(evs[2 * j].ms(evs[2 * j + 1]) for j in range(12))
    res.setdefault(kl, []).append(ts[len(ts) // 2])
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                     capture_output=True, text=True).stdout.strip()
print(f"{os.path.basename(os.environ.get('CQ_LIB', 'libcq.so'))} cfg={os.environ.get('CQ_WAVE_FUSED_CFG', 'default')}: parity {'ok' if ok else 'FAILED'}; "
      f"KL=8 median {min(res[8]):.4f} ms, KL=4 {res[4][0]:.4f} ms; clocks after: {clk}", flush=True)
