"""Fused wave pass: bit-exactness of the FMA (bounded) and exact forms
against one-step launches at 16384^2 and on odd shapes, then per-launch
timings of the KL = 8 / KL = 4 passes for several rows-per-warp settings
(CQ_FUSED_ROWS, read per launch).

    python scripts/r02/fused_ab.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402  (device memory only)

from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
K2, K4 = 2.0, 4.0


def view(t, h, w):
    v = N.CqView()
    v.ptr = t.data_ptr()
    v.alloc = N.box3((0, 0), (h, w))
    v.stride[:] = [h * w, w, 1]
    return v


def plain(a, b, h, w, steps, c):
    a, b = a.clone(), b.clone()
    torch.cuda.synchronize()   # torch's stream vs libcq's compute stream
    ext = N.box3((0, 0), (h, w))
    for _ in range(steps):
        N.call("cq_wave5", 0, 0, N.CQ_F32, ctypes.byref(view(a, h, w)), ctypes.byref(view(b, h, w)),
               ctypes.byref(view(b, h, w)), ctypes.byref(ext), ctypes.byref(ext), c, K2, K4)
        a, b = b, a
    return a, b


bound = torch.zeros(2, device="cuda", dtype=torch.float32)


def fused(a, b, h, w, kl, c, fast, in_rows=None, out_rows=None):
    ol, op = torch.full_like(a, float("nan")), torch.full_like(a, float("nan"))
    bound[0] = 1.0
    torch.cuda.synchronize()   # torch's stream vs libcq's compute stream
    ext = N.box3((0, 0), (h, w))
    in_rows = in_rows or (0, h)
    out_rows = out_rows or (0, h)
    N.call("cq_wave5_fused_bounded", 0, 0, N.CQ_F32, kl, ctypes.byref(view(a, h, w)), ctypes.byref(view(b, h, w)),
           ctypes.byref(view(ol, h, w)), ctypes.byref(view(op, h, w)), in_rows[0], in_rows[1], out_rows[0],
           out_rows[1], ctypes.byref(ext), c, K2, K4,
           ctypes.c_void_p(bound.data_ptr()) if fast else None, ctypes.c_void_p(bound.data_ptr() + 4))
    return ol, op


def same(x, y):
    return torch.equal(x.view(torch.int32), y.view(torch.int32))


ok = True
g = torch.Generator(device="cuda").manual_seed(11)
cases = [(16384, 16384, 0.25), (1000, 1024, 0.25), (517, 384, 0.3), (300, 4096, 0.25), (64, 128, 0.3),
         (2048, 2048, 0.3), (1100, 2176, 0.3), (40, 16384, 0.25), (16384, 256, 0.25)]
CFGS = [("1", "2", ""), ("1", "2", "7"), ("1", "2", "100"), ("1", "0", "3000")]
CFG_LIST = os.environ.get("PARITY_CFGS", "4,6").split(";")
for wpb, mp, env, cfg in ([] if os.environ.get("SKIP_PARITY") else
                          [c + (k,) for k in CFG_LIST for c in CFGS]):
    os.environ["CQ_WAVE_FUSED_CFG"] = cfg
    os.environ["CQ_FUSED_WPB"] = wpb
    os.environ["CQ_FUSED_MAP"] = mp
    if env:
        os.environ["CQ_FUSED_ROWS"] = env
    else:
        os.environ.pop("CQ_FUSED_ROWS", None)
    for (h, w, cc) in cases:
        if (env or wpb != "1") and h * w > 1 << 24:
            continue
        a = torch.rand((h, w), device="cuda", generator=g)
        b = torch.rand((h, w), device="cuda", generator=g)
        if cc != 0.25:
            a[:, :7] *= 1e-37
        for kl in ((4, 8) if cfg in ("4,6", "4,56") else (8,)):
            last, prev = plain(a, b, h, w, kl, cc)
            for fast in (False, True):
                fl, fp = fused(a, b, h, w, kl, cc, fast)
                torch.cuda.synchronize()
                r = same(fl, last) and same(fp, prev)
                ok &= r
                if not r:
                    d = (fl != last).nonzero()
                    print(f"MISMATCH rows={env or 'auto'} {h}x{w} c={cc} KL={kl} fast={fast}: {d[:5].tolist()}",
                          flush=True)
            lo, hi = h // 4, 3 * h // 4
            if hi - lo > 2 * kl + 2:
                fl, fp = fused(a, b, h, w, kl, cc, True, (lo, hi), (lo + kl, hi - kl))
                torch.cuda.synchronize()
                s = slice(lo + kl, hi - kl)
                r = same(fl[s], last[s]) and same(fp[s], prev[s])
                ok &= r
                if not r:
                    print(f"MISMATCH slab rows={env or 'auto'} {h}x{w} KL={kl}", flush=True)
    print(f"cfg={cfg} wpb={wpb} map={mp} rows={env or 'auto'}: parity {'ok' if ok else 'FAILED'}", flush=True)
for k in ("CQ_FUSED_ROWS", "CQ_WAVE_FUSED_CFG", "CQ_FUSED_WPB", "CQ_FUSED_MAP"):
    os.environ.pop(k, None)


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
t = [torch.rand((h, w), device="cuda", generator=g) for _ in range(4)]
vs = [view(x, h, w) for x in t]
ext = N.box3((0, 0), (h, w))
e0, e1 = Ev(), Ev()
geo = (ctypes.c_int64 * 4)()
def sweep(runs, reps=7, per=4):
    """Interleaved timing: every rep runs every config (env set per launch,
    2 warm-up + ``per`` timed launches each, one event pair per launch); the
    median per config is reported, so clock drift hits all configs alike."""
    times = {r: [] for r in runs}
    evs = [Ev() for _ in range(2 * per)]
    for _rep in range(reps):
        for r in runs:
            kl, env = r[0], dict(r[1])
            for k in ("CQ_FUSED_WPB", "CQ_FUSED_MAP", "CQ_FUSED_ROWS", "CQ_WAVE_FUSED_CFG"):
                os.environ.pop(k, None)
            os.environ.update(env)
            for i in range(2 + per):
                s_, d_ = (vs[0], vs[1]), (vs[2], vs[3])
                if i % 2:
                    s_, d_ = d_, s_
                bound[0] = 1.0
                if i >= 2:
                    evs[2 * (i - 2)].record()
                N.call("cq_wave5_fused_bounded", 0, 0, N.CQ_F32, kl, ctypes.byref(s_[0]), ctypes.byref(s_[1]),
                       ctypes.byref(d_[0]), ctypes.byref(d_[1]), 0, h, 0, h, ctypes.byref(ext), 0.25, K2, K4,
                       ctypes.c_void_p(bound.data_ptr()), ctypes.c_void_p(bound.data_ptr() + 4))
                if i >= 2:
                    evs[2 * (i - 2) + 1].record()
            N.call("cq_stream_synchronize", 0, 0)
            times[r] += [evs[2 * j].ms(evs[2 * j + 1]) for j in range(per)]
    for r in runs:
        kl, env = r[0], dict(r[1])
        os.environ.update(env)
        N.call("cq_wave5_fused_geometry", 0, N.CQ_F32, kl, h, w, geo)
        t = sorted(times[r])
        ms = t[len(t) // 2]
        print(f"KL={kl} {env or 'default'} geo={list(geo)} recompute={1 - h * w / geo[3]:.4f}: median {ms:.4f} ms "
              f"(min {t[0]:.4f}, max {t[-1]:.4f}, n={len(t)}) = {12 * h * w * kl / ms / 1e6:.0f} GB/s effective",
              flush=True)
        for k in env:
            os.environ.pop(k, None)


def clocks():
    import subprocess
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                               "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except OSError:
        return "?"


RUNS8 = [(8, ()), (8, (("CQ_WAVE_FUSED_CFG", "4,56"),)), (8, (("CQ_WAVE_FUSED_CFG", "4,59"),))]
RUNS4 = [(4, ()), (4, (("CQ_WAVE_FUSED_CFG", "4,56"),))]
print("clocks before:", clocks(), flush=True)
sweep(RUNS8)
print("clocks:", clocks(), flush=True)
sweep(RUNS4)
print("clocks after:", clocks(), flush=True)
print("ALL OK" if ok else "FAILED", flush=True)
sys.exit(0 if ok else 1)
