"""A/B of the fused wave pass's segment length: automatic (wave-quantisation
aware, default) vs a fixed CQ_FUSED_SEG.  Times back-to-back launches of
cq_wave5_fused on one GPU at several slab heights (wall clock over many
queued launches, one synchronize).

    python scripts/fused_seg_ab.py            # runs both arms as subprocesses
"""
import ctypes
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def arm():
    import torch
    from paper_2505_06022_b200 import _native as N
    N.call("cq_init_device", 0)
    w = 16384
    out = []
    for h in (16384, 8192, 4096, 1024, 512):
        t = [torch.rand((h, w), device="cuda") for _ in range(4)]
        torch.cuda.synchronize()

        def view(x):
            v = N.CqView()
            v.ptr = x.data_ptr()
            v.alloc = N.box3((0, 0), (h, w))
            v.stride[:] = [h * w, w, 1]
            return v
        vs = [view(x) for x in t]
        ext = N.box3((0, 0), (h, w))
        for kl in (8, 4):
            def go(n):
                for _ in range(n):
                    N.call("cq_wave5_fused", 0, 0, N.CQ_F32, kl, ctypes.byref(vs[0]), ctypes.byref(vs[1]),
                           ctypes.byref(vs[2]), ctypes.byref(vs[3]), 0, h, 0, h, ctypes.byref(ext), 0.25, 2.0, 4.0)
                N.call("cq_stream_synchronize", 0, 0)
            go(3)
            reps = max(10, int(2e4 // h))
            t0 = time.perf_counter()
            go(reps)
            dt = (time.perf_counter() - t0) / reps
            out.append(f"h={h:6d} KL={kl} {dt * 1e3:8.3f} ms/pass  {h * w * kl / dt / 1e9:8.1f} Gcell-steps/s")
        del t, vs
    print("\n".join(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "arm":
        arm()
        sys.exit(0)
    for label, env in (("auto", {}), ("fixed RB (CQ_FUSED_SEG=256)", {"CQ_FUSED_SEG": "256"}),
                       ("fixed 128", {"CQ_FUSED_SEG": "128"})):
        print(f"== {label}", flush=True)
        subprocess.run([sys.executable, __file__, "arm"], env={**os.environ, **env}, check=True)
