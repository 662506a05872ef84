"""GPU check of cq_wave5_fused (KL steps per pass) against KL launches of
cq_wave5: bit-identical on full grids and on row slabs, then timing at 16384^2."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402  (device memory only)

from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
C, K2, K4 = 0.25, 2.0, 4.0


def view(t, h, w):
    v = N.CqView()
    v.ptr = t.data_ptr()
    v.alloc = N.box3((0, 0), (h, w))
    v.stride[:] = [h * w, w, 1]
    return v


def plain(a, b, h, w, steps, rows=None, C=C):
    """steps one-step launches, ping-pong in place; returns (X(t+steps), X(t+steps-1))."""
    a, b = a.clone(), b.clone()
    ext = N.box3((0, 0), (h, w))
    box = N.box3((0, 0), (h, w)) if rows is None else N.box3((rows[0], 0), (rows[1], w))
    for _ in range(steps):
        N.call("cq_wave5", 0, 0, N.CQ_F32, ctypes.byref(view(a, h, w)), ctypes.byref(view(b, h, w)),
               ctypes.byref(view(b, h, w)), ctypes.byref(box), ctypes.byref(ext), C, K2, K4)
        a, b = b, a
    return a, b


def fused(a, b, h, w, kl, in_rows, out_rows, C=C):
    ol, op = torch.full_like(a, float("nan")), torch.full_like(a, float("nan"))
    ext = N.box3((0, 0), (h, w))
    N.call("cq_wave5_fused", 0, 0, N.CQ_F32, kl, ctypes.byref(view(a, h, w)), ctypes.byref(view(b, h, w)),
           ctypes.byref(view(ol, h, w)), ctypes.byref(view(op, h, w)), in_rows[0], in_rows[1],
           out_rows[0], out_rows[1], ctypes.byref(ext), C, K2, K4)
    return ol, op


def same(x, y):
    return torch.equal(x.view(torch.int32), y.view(torch.int32))


ok = True
g = torch.Generator(device="cuda").manual_seed(7)
for (h, w, cc) in [(1000, 1024, 0.25), (517, 384, 0.3), (300, 4096, 0.25), (64, 128, 0.3), (2048, 2048, 0.3),
                   (1100, 2176, 0.3)]:
    a = torch.rand((h, w), device="cuda", generator=g)
    b = torch.rand((h, w), device="cuda", generator=g)
    if cc != 0.25:
        a[:, :7] *= 1e-37  # subnormal neighbourhoods: c * lap must round on its own
    for kl in (4, 8):
        last, prev = plain(a, b, h, w, kl, C=cc)
        fl, fp = fused(a, b, h, w, kl, (0, h), (0, h), C=cc)
        torch.cuda.synchronize()
        r = same(fl, last) and same(fp, prev)
        ok &= r
        print(f"full {h}x{w} c={cc} KL={kl}: {'bit-identical' if r else 'MISMATCH'}", flush=True)
        if not r:
            d = (fl != last).nonzero()
            print("   first mismatches (last):", d[:5].tolist(), flush=True)
        # a slab: inputs rows [lo, hi) only, outputs inside the trapezoid
        lo, hi = h // 4, 3 * h // 4
        if hi - lo > 2 * kl + 2:
            fl, fp = fused(a, b, h, w, kl, (lo, hi), (lo + kl, hi - kl), C=cc)
            torch.cuda.synchronize()
            r = same(fl[lo + kl:hi - kl], last[lo + kl:hi - kl]) and same(fp[lo + kl:hi - kl], prev[lo + kl:hi - kl])
            ok &= r
            print(f"slab {h}x{w} rows [{lo},{hi}) KL={kl}: {'bit-identical' if r else 'MISMATCH'}", flush=True)

# huge values: the per-warp guard must switch to the separate-product tree
# (FMA-folded 4u / 2u would not overflow where the tree does)
for (h, w, row) in [(600, 1024, 0), (600, 1024, 333), (300, 2176, 150)]:
    a = torch.rand((h, w), device="cuda", generator=g)
    b = torch.rand((h, w), device="cuda", generator=g)
    a[row, 100:140] = 1.5e38
    b[row + 3, 500:520] = -2.0e38
    a[row + 7, 700] = float("inf")
    for kl in (4, 8):
        last, prev = plain(a, b, h, w, kl, C=0.3)
        fl, fp = fused(a, b, h, w, kl, (0, h), (0, h), C=0.3)
        torch.cuda.synchronize()
        r = same(fl, last) and same(fp, prev)
        ok &= r
        print(f"huge values at row {row} {h}x{w} KL={kl}: {'bit-identical' if r else 'MISMATCH'}", flush=True)

# timing at the BASELINE tile
h = w = 16384
a = torch.rand((h, w), device="cuda", generator=g)
b = torch.rand((h, w), device="cuda", generator=g)
a2, b2 = torch.empty_like(a), torch.empty_like(a)
ext = N.box3((0, 0), (h, w))
box = N.box3((0, 0), (h, w))
va, vb, va2, vb2 = (view(t, h, w) for t in (a, b, a2, b2))


class Ev:
    """cq timing event on the compute stream (the kernels' stream, not torch's)."""
    def __init__(self):
        h = ctypes.c_uint64()
        N.call("cq_event_create", 0, 1, ctypes.byref(h))
        self.h = h.value

    def record(self):
        N.call("cq_event_record", ctypes.c_uint64(self.h), 0, 0)

    def elapsed_time(self, other):
        ms = ctypes.c_float()
        N.call("cq_event_elapsed_ms", ctypes.c_uint64(self.h), ctypes.c_uint64(other.h), ctypes.byref(ms))
        return ms.value


def sync():
    N.call("cq_stream_synchronize", 0, 0)


ev = [Ev(), Ev()]
steps = 96
for rep in range(2):
    torch.cuda.synchronize()
    sync()
    ev[0].record()
    x, y = va, vb
    for _ in range(steps):
        N.call("cq_wave5", 0, 0, N.CQ_F32, ctypes.byref(x), ctypes.byref(y), ctypes.byref(y), ctypes.byref(box),
               ctypes.byref(ext), C, K2, K4)
        x, y = y, x
    ev[1].record()
    sync()
    ms = ev[0].elapsed_time(ev[1])
    print(f"plain {steps} steps: {ms:.2f} ms = {12 * h * w * steps / ms / 1e6:.0f} GB/s effective", flush=True)
for kl in (4, 8):
    for rep in range(2):
        torch.cuda.synchronize()
        sync()
        ev[0].record()
        src, dst = (va, vb), (va2, vb2)
        for _ in range(steps // kl):
            N.call("cq_wave5_fused", 0, 0, N.CQ_F32, kl, ctypes.byref(src[0]), ctypes.byref(src[1]), ctypes.byref(dst[0]),
                   ctypes.byref(dst[1]), 0, h, 0, h, ctypes.byref(ext), C, K2, K4)
            src, dst = dst, src
        ev[1].record()
        sync()
        ms = ev[0].elapsed_time(ev[1])
        print(f"fused KL={kl} {steps} steps: {ms:.2f} ms = {12 * h * w * steps / ms / 1e6:.0f} GB/s effective "
              f"({16 * h * w * (steps // kl) / ms / 1e6:.0f} GB/s of 16 B/cell/pass)", flush=True)
# FLOAT64: the fused double kernel (two doubles per lane) against one-step launches
def view64(t, h, w):
    return view(t, h, w)


for (h, w) in [(517, 384), (300, 1024)]:
    a = torch.rand((h, w), device="cuda", generator=g, dtype=torch.float64)
    b = torch.rand((h, w), device="cuda", generator=g, dtype=torch.float64)
    for kl in (4, 8):
        x, y = a.clone(), b.clone()
        ext = N.box3((0, 0), (h, w))
        box = N.box3((0, 0), (h, w))
        for _ in range(kl):
            N.call("cq_wave5", 0, 0, N.CQ_F64, ctypes.byref(view(x, h, w)), ctypes.byref(view(y, h, w)),
                   ctypes.byref(view(y, h, w)), ctypes.byref(box), ctypes.byref(ext), 0.3, K2, K4)
            x, y = y, x
        ol, op = torch.full_like(a, float("nan")), torch.full_like(a, float("nan"))
        N.call("cq_wave5_fused", 0, 0, N.CQ_F64, kl, ctypes.byref(view(a, h, w)), ctypes.byref(view(b, h, w)),
               ctypes.byref(view(ol, h, w)), ctypes.byref(view(op, h, w)), 0, h, 0, h, ctypes.byref(ext), 0.3, K2, K4)
        torch.cuda.synchronize()
        sync()
        r = torch.equal(ol.view(torch.int64), x.view(torch.int64)) and torch.equal(op.view(torch.int64), y.view(torch.int64))
        ok &= r
        print(f"float64 {h}x{w} KL={kl}: {'bit-identical' if r else 'MISMATCH'}", flush=True)
h = w = 16384
a = torch.rand((h, w), device="cuda", generator=g, dtype=torch.float64)
b = torch.rand((h, w), device="cuda", generator=g, dtype=torch.float64)
a2, b2 = torch.empty_like(a), torch.empty_like(a)
va, vb, va2, vb2 = (view(t, h, w) for t in (a, b, a2, b2))
ext = N.box3((0, 0), (h, w))
for kl in (4, 8):
    torch.cuda.synchronize()
    sync()
    ev[0].record()
    src, dst = (va, vb), (va2, vb2)
    for _ in range(96 // kl):
        N.call("cq_wave5_fused", 0, 0, N.CQ_F64, kl, ctypes.byref(src[0]), ctypes.byref(src[1]), ctypes.byref(dst[0]),
               ctypes.byref(dst[1]), 0, h, 0, h, ctypes.byref(ext), 0.25, K2, K4)
        src, dst = dst, src
    ev[1].record()
    sync()
    ms = ev[0].elapsed_time(ev[1])
    print(f"float64 fused KL={kl} 96 steps: {ms:.2f} ms = {24 * h * w * 96 / ms / 1e6:.0f} GB/s effective (24 B/cell/step)",
          flush=True)
print("ALL OK" if ok else "FAILED", flush=True)
sys.exit(0 if ok else 1)
