#!/usr/bin/env python
"""BASELINE benchmark: "GB/s (or GFLOP/s) per kernel at 1/2/4/8 B200, %
roofline; J/iteration vs SM clock" (BASELINE.json).

Headline workload = BASELINE configs[1]: the 2-D wave_sim 5-point stencil,
fp32, 100 time steps, neighborhood(1,1) halo exchange, weak-scaled at
16384 x 16384 cells per GPU (global 16384*N x 16384).  One bench *step* is
one full 100-time-step simulation through the reference-shaped API:
Buffer/Task/TaskGraph -> generate_commands -> B200 executor.

* value     -- device-resident: the plan re-executed on data already in HBM
               (Session.execute(upload=False)), CUDA events, max over ranks.
* e2e       -- the public API with host buffers: ``run_batch`` of K
               simulations, each uploading its inputs from pinned host memory
               (H2D inside the timed region) and reading both result fields
               back, three in flight so the PCIe directions and the SMs overlap;
               the one-at-a-time ``run(plan)`` number is reported as e2e.sync.
* roofline  -- the dominant kernel: the temporally blocked wave pass
               (cq_wave5_fused, 8 time steps per HBM pass: 16 algorithmic
               bytes per cell per launch) -- or the one-step kernel (12 B/cell)
               with CQ_WAVE_FUSE=0 -- over its CUDA-event launch time, against
               MEASURED_PEAKS.json hbm_gbs.  ``value`` keeps the SURVEY unit
               (12 B per cell per time step), so with temporal blocking it can
               exceed the HBM peak.
* kernels   -- the other BASELINE workloads at this N (SAXPY, N-body, sgemm).
* energy    -- NVML J/iteration per kernel at the running SM clock.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIZE = 16384
WAVE_STEPS = 100
SWEEP_SECONDS = 1.0   # NVML energy window per clock point
C = 0.25


def _baseline_metric():
    """BASELINE.json's metric string, printed verbatim by BOTH arms (the
    driver pairs the b200 and reference lines by metric, unit and
    higher_is_better)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as fh:
            return json.load(fh)["metric"]
    except (OSError, KeyError, ValueError):
        return "GB/s (or GFLOP/s) per kernel at 1/2/4/8 B200, % roofline; J/iteration vs SM clock"


METRIC = _baseline_metric()
UNIT = "GB/s"
# what `value` measures under that metric (both arms)
METRIC_DETAIL = ("wave_sim 5-point stencil, 12 B x cells x time steps / time (SURVEY.md §8d: read u, "
                 "read u_prev, write u_next per cell per time step)")


def headline_config(size, world, wave_steps):
    """The headline workload (BASELINE configs[1]), identical in both arms."""
    return {"workload": f"wave_sim 2-D 5-point stencil {size}x{size} fp32 per GPU (global {size * world}x{size}), "
                        f"{wave_steps} time steps per bench step, neighborhood(1,1) halo exchange",
            "metric_detail": METRIC_DETAIL,
            "parallelism": f"dp{world} (row slabs, one rank per GPU)",
            "l2": "inputs 2 GiB/GPU >> 126 MB L2 (no flush needed)",
            "init": "Gaussian pulse (SURVEY.md §8d)"}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ distributed

class Dist:
    def __init__(self, gpus):
        self.world = _env_int("WORLD_SIZE", 1)
        self.rank = _env_int("RANK", 0)
        self.local_rank = _env_int("LOCAL_RANK", 0)
        self.gpus = gpus
        self.torch = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            import datetime
            torch.cuda.set_device(self.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank),
                                    timeout=datetime.timedelta(seconds=300))
            self.torch = torch
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([float(x)], device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def min(self, x):
        return -self.max(-x)

    def sum(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([float(x)], device="cuda")
        self.dist.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# -------------------------------------------------------------- wave program

def wave_inputs(h, w, rows, both=True):
    """Gaussian pulse, written only for the rows this rank
    touches (the rest of the big host arrays stays virtual); ``both=False``
    returns (u0, None)."""
    from paper_2505_06022_b200 import executor as E
    from paper_2505_06022_b200.region import Box
    box = Box((rows[0], 0), (rows[1], w))
    u0 = E.pinned_empty((h, w), np.float32, box)
    up0 = E.pinned_empty((h, w), np.float32, box) if both else None
    j = np.arange(w, dtype=np.float64)[None, :] - w / 2
    jj = j * j
    s2 = 2 * (w / 16.0) ** 2
    for r0 in range(rows[0], rows[1], 1024):  # row blocks keep host temporaries small
        r1 = min(r0 + 1024, rows[1])
        i = np.arange(r0, r1, dtype=np.float64)[:, None] - h / 2
        u0[r0:r1] = np.exp(-(i * i + jj) / s2).astype(np.float32)
        if up0 is not None:
            up0[r0:r1] = u0[r0:r1]
    return u0, up0


def pulse_field(h, w):
    """The same Gaussian pulse as ``wave_inputs`` as a plain host array (the
    CPU arms)."""
    out = np.empty((h, w), np.float32)
    j = np.arange(w, dtype=np.float64)[None, :] - w / 2
    jj = j * j
    s2 = 2 * (w / 16.0) ** 2
    for r0 in range(0, h, 1024):
        r1 = min(r0 + 1024, h)
        i = np.arange(r0, r1, dtype=np.float64)[:, None] - h / 2
        out[r0:r1] = np.exp(-(i * i + jj) / s2).astype(np.float32)
    return out


def sm_count():
    try:
        import torch
        return torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:  # noqa: BLE001
        return 148


def bench_wave(args, dist, placement, peaks):
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import executor as E
    from paper_2505_06022_b200 import workloads as W
    from paper_2505_06022_b200.region import Box

    world, rank = dist.world, dist.rank
    H, Wd, steps = args.size * world, args.size, args.wave_steps
    lo, hi = rank * args.size, (rank + 1) * args.size
    rows = (max(lo - 1, 0), min(hi + 1, H))
    # u0 = up0 = the pulse: one host array initialises both
    # buffers, so it crosses PCIe once per simulation (executor: device copy)
    u0, _ = wave_inputs(H, Wd, rows, both=False)
    prog = W.wave_program(H, Wd, steps=steps, kind="float32", c=C, u0=u0, up0=u0)
    t0 = time.perf_counter()
    plan = cq.generate_commands(prog.graph(), world)
    plan_s = time.perf_counter() - t0

    # ---- device-resident value ------------------------------------------
    sess = E.Session(plan, placement, trace=True)
    if sess.chains:
        ch = sess.chains[0]
        execution = (f"temporal blocking (fusion.py): {len(ch.blocks)} out-of-place passes "
                     f"({' + '.join(f'{sum(b.kl == k for b in ch.blocks)} x KL{k}' for k in sorted({b.kl for b in ch.blocks}, reverse=True))}) of cq_wave5_fused + "
                     f"{len(ch.plain)} one-step launches per 100 steps; KL-row halo exchange per pass "
                     f"(bit-identical to the per-step plan)")
    else:
        execution = "one cq_wave5 launch per time step (CQ_WAVE_FUSE=0 or not fusable)"
    sess.execute(upload=True)
    sess.synchronize()
    sess.recycle()
    # one traced replay: per-launch CUDA-event times of every kernel
    sess.execute(upload=False)
    sess.synchronize()
    # the dominant kernel: the temporally blocked KL=4 pass when the chain is
    # fused (16 algorithmic B/cell per launch: read X(t), X(t-1), write
    # X(t+4), X(t+3)), else the one-step kernel (12 B/cell)
    totals = {}
    for x in sess.launch_log:
        if x[0].startswith("wave5"):
            totals[x[0]] = totals.get(x[0], 0) + x[1]
    dom_kind = max(totals, key=totals.get)   # most cells: wave5_fused8 / _fused4 / wave5
    bpc = 16 if dom_kind != "wave5" else 12
    wave_launches = [x for x in sess.launch_log if x[0] == dom_kind]
    launches_per_replay = len(sess.launch_log)
    # dominant launches only: at N > 1 the halo-row launches run concurrently
    # on the boundary stream, so summing every launch would double-count time
    dom_launch = max(wave_launches, key=lambda x: x[1])
    dominant = [x for x in wave_launches if x[1] == dom_launch[1]]
    kern_ms = sum(sess.elapsed_ms(a, b) for _k, _c, _d, _s, a, b in dominant)
    kern_bytes = sum(bpc * cells for _k, cells, *_ in dominant)
    sess.recycle()
    timing_source = "stream-traced replay"
    if not args.no_graph:
        def select(log):
            return [x for x in log if x[0] == dom_kind and x[1] == dom_launch[1]]
        g = graph_launch_times(sess, 2, select)
        if g and dom_kind in g:
            kern_bytes, kern_ms = bpc * g[dom_kind][0], g[dom_kind][1]
            timing_source = "timed CUDA-graph replay (event-record nodes)"
    # the timed replays run as one CUDA graph per rank (kernels, copies and
    # NCCL groups captured once), so no per-command host dispatch remains
    replay_mode = "cuda_graph"
    if args.no_graph:
        replay_mode = "stream"
    else:
        try:
            sess.capture()
        except Exception as exc:  # noqa: BLE001
            replay_mode = f"stream (graph capture failed: {exc})"[:200]
            sess.synchronize()
            sess.recycle()
    graph = replay_mode == "cuda_graph"

    def replay_once():
        if graph:
            sess.replay(1)
        else:
            sess.execute(upload=False)

    for _ in range(args.warmup):
        replay_once()
        sess.synchronize()
        if not graph:
            sess.recycle()
    dist.barrier()
    dev = placement.devices[0]
    with ClockSampler(dev) as clocks:
        m0 = sess.mark()
        for _ in range(args.steps):
            replay_once()
        m1 = sess.mark()
        sess.synchronize()
    dev_ms = max(sess.elapsed_ms(m0[d], m1[d]) for d in sess.devices)
    gpu_launches = launches_per_replay * args.steps
    sess.recycle()
    energy = energy_loop(sess, dist, dev_ms / args.steps, 1.5) if args.energy else None
    if energy and "j_per_iter" in energy:
        energy["j_per_time_step"] = energy["j_per_iter"] / steps
        energy["gb_per_joule"] = 12 * H * Wd * steps / 1e9 / energy["j_per_iter"] / world
    sess.close()
    dev_ms = dist.max(dev_ms)
    cells = H * Wd * steps * args.steps
    value = 12 * cells / (dev_ms / 1e3) / 1e9
    steps_per_launch = {"wave5_fused8": 8, "wave5_fused4": 4}.get(dom_kind, 1)
    kern_s = kern_ms / 1e3
    cells_launch = kern_bytes / bpc   # output cells of the timed launches
    clk = clocks.summary()

    # ---- end to end through the public API, host buffers ------------------
    # run_batch: every simulation uploads its inputs from pinned host memory
    # and reads both result fields back; two simulations are in flight, so
    # one's read-back, the next one's upload and the kernels overlap.  The
    # one-at-a-time run(plan) is reported beside it ("sync").
    gather = "root" if world == 1 else "local"
    out_box = Box((lo, 0), (hi, Wd))
    depth = int(os.environ.get("CQ_BATCH_DEPTH", "3"))
    outs = [{"u": E.pinned_empty((H, Wd), np.float32, out_box),
             "up": E.pinned_empty((H, Wd), np.float32, out_box)} for _ in range(depth)]
    # warm-up: two full turns of the sessions (the first run_batch after the
    # device-resident leg measured 95-220 ms per job on some boxes, the
    # following ones the PCIe duplex floor; scripts/r02/e2e_diag*.py)
    E.run_batch(plan, [(None, outs[k % depth]) for k in range(max(2 * depth, args.warmup))], gather=gather,
                depth=depth)
    # three timed batches of K simulations each, the median reported (a box
    # has shown one-off batches at 2-3x its usual time; all three are listed)
    batches_s = []
    for _rep in range(3):
        dist.barrier()
        h2d0 = E.STATS["h2d_bytes"]
        t0 = time.perf_counter()
        batch = E.run_batch(plan, [(None, outs[k % depth]) for k in range(args.steps)], gather=gather, depth=depth)
        batches_s.append(dist.max(time.perf_counter() - t0))
        h2d = int(dist.sum((E.STATS["h2d_bytes"] - h2d0) / args.steps))   # bytes that crossed PCIe per simulation
    e2e_s = sorted(batches_s)[1]
    e2e = 12 * cells / e2e_s / 1e9
    res_buffers = batch[-1]
    E.run(plan, gather=gather, out=outs[0], trace=False)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        E.run(plan, gather=gather, out=outs[0], trace=False)
    sync_s = dist.max(time.perf_counter() - t0)
    d2h = int(dist.sum(2 * (hi - lo) * Wd * 4))
    newest = W.wave_result_buffer(steps)
    field = res_buffers[newest][lo:hi]
    finite = bool(np.isfinite(field).all())

    roofline = wave_roofline(dom_kind, dom_launch[1], len(dominant), cells_launch, kern_s, steps_per_launch,
                             bpc, clk, peaks, dist, placement.devices[0], Wd, timing_source)
    # the PCIe copies bound e2e: the floor for this rank's bytes per simulation
    b_in, b_out = h2d // world, d2h // world
    link = pcie_floor(placement.devices[0], pattern=(b_in - b_in % 16, b_out - b_out % 16))
    link["floor_model_ms"] = max(b_in / (link["h2d_gbs"] * 1e9), b_out / (link["d2h_gbs"] * 1e9),
                                 (b_in + b_out) / (link["duplex_gbs"] * 1e9)) * 1e3
    link["floor_ms_per_step"] = link["pattern_ms"]
    link["note"] = ("e2e moves every simulation's inputs in and both fields out over PCIe; floor = one "
                    "simulation's own H2D and D2H bytes copied concurrently with nothing else running "
                    "(pattern_ms, per rank); floor_model_ms = the slowest of h2d bytes / h2d rate, d2h bytes "
                    "/ d2h rate and both / the 1:1 duplex rate")

    return {
        "value": value, "ms_per_step": dev_ms / args.steps, "plan_s": plan_s,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3 / args.steps, "gather": gather, "finite": finite, "pcie": link,
                "batches_ms_per_step": [b * 1e3 / args.steps for b in batches_s],
                "timing": "median of three timed run_batch calls of --steps simulations each",
                "api": f"executor.run_batch (depth {depth}: upload, kernels and read-back of simulations overlap)",
                "sync": {"value": 12 * cells / sync_s / 1e9, "ms_per_step": sync_s * 1e3 / args.steps,
                         "api": "executor.run (one simulation at a time)"}},
        "roofline": roofline,
        "clocks": clk,
        "gpu_launches": gpu_launches,
        "replay": replay_mode,
        "energy": energy,
        "execution": execution,
        "H": H, "W": Wd,
    }


def pcie_floor(device, nbytes=1 << 30, pattern=None):
    """The e2e leg's own roofline: H2D, D2H and concurrent H2D + D2H of
    ``nbytes`` each between page-locked host memory and the GPU, and, with
    ``pattern`` = (h2d bytes, d2h bytes), one simulation's actual transfers
    issued concurrently with nothing else running (best of 3 each, through
    libcq's copy streams)."""
    import ctypes
    from paper_2505_06022_b200 import _native as N, executor as E
    up, down = pattern or (nbytes, nbytes)
    n_in, n_out = max(nbytes, up), max(nbytes, down)
    src = E.pinned_empty((n_in // 4,), np.float32)
    dst = E.pinned_empty((n_out // 4,), np.float32)
    src[:] = 1.0
    d1, d2 = ctypes.c_void_p(), ctypes.c_void_p()
    N.call("cq_malloc", device, n_in, ctypes.byref(d1))
    N.call("cq_malloc", device, n_out, ctypes.byref(d2))
    lanes = (N.STREAM_LANE0, N.STREAM_LANE0 + 1)

    def sync():
        for st in lanes:
            N.call("cq_stream_synchronize", device, st)
    best = {}
    sizes = {"h2d": (nbytes, 0), "d2h": (0, nbytes), "duplex": (nbytes, nbytes)}
    if pattern:
        sizes["pattern"] = (up, down)
    try:
        for name, (b_in, b_out) in sizes.items():
            for _ in range(3):
                sync()
                t0 = time.perf_counter()
                if b_in:
                    N.call("cq_copy_h2d", device, lanes[0], d1, ctypes.c_void_p(src.ctypes.data), b_in)
                if b_out:
                    N.call("cq_copy_d2h", device, lanes[1], ctypes.c_void_p(dst.ctypes.data), d2, b_out)
                sync()
                dt = time.perf_counter() - t0
                best[name] = min(best.get(name, 1e9), dt)
    finally:
        N.call("cq_free", device, d1)
        N.call("cq_free", device, d2)
    out = {"bytes_each_way": nbytes, "h2d_gbs": nbytes / best["h2d"] / 1e9, "d2h_gbs": nbytes / best["d2h"] / 1e9,
           "duplex_gbs": 2 * nbytes / best["duplex"] / 1e9}
    if pattern:
        out["pattern_bytes"] = [up, down]
        out["pattern_ms"] = best["pattern"] * 1e3
    return out


def wave_roofline(kind, cells_per_launch, launches, cells_timed, kern_s, levels, bpc, clk, peaks, dist, device,
                  width, timing_source):
    """Roofline of the dominant wave kernel against the resource that binds it.

    * one-step kernel / KL=4 pass: HBM.  achieved = the kernel's own minimum
      traffic (12 B/cell one-step, 16 B/cell per fused pass: read X(t),
      X(t-1), write two levels) over its CUDA-event launch time.
    * KL=8 pass: FP32 pipe / issue (ncu: FMA pipe and issue ~70% busy, DRAM
      below peak).  achieved = USEFUL FP32 lane-ops -- 7 per cell per level
      (n+s, +w, +e, fma(-4,u,.), fma(2,u,-p), c*lap, +), recompute
      of halo columns / rows not counted -- over the launch time; peak =
      SMs x 128 lanes x the SM clock observed in the timed region.  The DRAM
      fraction (ncu bytes), the recompute share (launch geometry) and the
      12-B/cell/step rate (``effective_gbs``) are reported beside it."""
    from paper_2505_06022_b200 import _native as N
    import ctypes
    hbm = peaks[0]["hbm_gbs"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"{kind}_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            t = json.load(fh)
        if t.get("cells"):
            traffic = t["dram_bytes"] / t["cells"] * cells_per_launch
    effective = dist.min(12 * levels * cells_timed / kern_s / 1e9)
    own = dist.min(bpc * cells_timed / kern_s / 1e9)
    names = {"wave5_fused8": "wave5_fused_kernel<float,8,4,6,1> (8 time steps per pass; one-warp blocks, "
                             "224-row strip-minor pieces)",
             "wave5_fused4": "wave5_fused_kernel<float,4,4,6,1> (4 time steps per pass; 24-row pieces)"}
    out = {"kernel": names.get(kind, "wave5_rows_kernel<float,32>"), "cells_per_launch": cells_per_launch,
           "launches": launches, "time_steps_per_launch": levels, "launch_timing": timing_source,
           "effective_gbs": effective, "effective_note": "12 B x cells x time steps per launch / launch time "
                                                          "(SURVEY §8d unit; not a traffic rate)",
           "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                           f"(profiles/{kind}_traffic.json)"}
    if kind != "wave5_fused8":
        out.update({"bound": "hbm", "achieved": own, "peak": hbm, "unit": "GB/s", "frac": own / hbm,
                    "traffic": traffic, "algorithmic_bytes_per_cell": bpc,
                    "peak_source": peaks[1] + " hbm_gbs (torch copy)"})
        return out
    sms = sm_count()
    mhz = clk.get("sm_mhz") or peaks[0].get("sm_max_mhz", 1965.0)
    mx = peaks[0].get("sm_max_mhz", 1965.0)
    ops = 7 * levels * cells_timed / kern_s / 1e9        # useful G lane-ops/s
    ops = dist.min(ops)
    peak = sms * 128 * mhz / 1e3                          # G lane-ops/s at the observed clock
    geo = (ctypes.c_int64 * 4)()
    try:
        N.call("cq_wave5_fused_geometry", device, N.CQ_F32, levels, cells_per_launch // width, width, geo)
        computed = geo[3]
        recompute = 1.0 - cells_per_launch / computed
        geometry = {"rows_per_piece": geo[0], "blocks": geo[1], "warps": geo[2], "computed_cells_per_level": computed}
    except Exception as exc:  # noqa: BLE001
        recompute, geometry = None, {"error": str(exc)[:200]}
    launch_s = kern_s * cells_per_launch / cells_timed   # average launch duration
    dram_gbs = traffic / launch_s / 1e9 if traffic else None
    out.update({"bound": "fp32_issue", "achieved": ops, "peak": peak, "unit": "G FP32 lane-ops/s",
                "frac": ops / peak, "traffic": traffic,
                "peak_definition": f"{sms} SMs x 128 FP32 lanes x {mhz:.0f} MHz (median SM clock in the timed "
                                   "region), one lane-op per lane per cycle",
                "peak_at_max_clock": sms * 128 * mx / 1e3, "frac_at_max_clock": ops / (sms * 128 * mx / 1e3),
                "useful_ops_per_cell_level": 7, "recompute_share": recompute, "geometry": geometry,
                "dram": {"achieved_gbs": dram_gbs, "peak_gbs": hbm,
                         "frac": dram_gbs / hbm if dram_gbs else None,
                         "kernel_min_bytes_per_cell": bpc, "achieved_min_bytes_gbs": own}})
    return out


# -------------------------------------------------------- other BASELINE kernels

def graph_launch_times(sess, reps, select=None):
    """Per-launch CUDA-event durations of the dominant kernels, read from
    ``reps`` replays of a timed CUDA graph (event-record nodes around every
    launch): the launches run exactly as in the timed region, back to back
    with no host dispatch between them.  Returns {kind: [cells, ms, launches]}
    over the launches ``select(log)`` keeps (default: all), or None when the
    graph cannot be captured (then the caller keeps its stream-traced times)."""
    try:
        sess.capture(timed=True)
    except Exception:  # noqa: BLE001
        sess.synchronize()
        sess.recycle()
        return None
    sess.replay(1)
    sess.synchronize()
    per_kind = {}
    for _ in range(reps):
        sess.replay(1)
        sess.synchronize()
        log = sess.graph_log if select is None else select(sess.graph_log)
        for kind, cells, _d, _s, a, b in log:
            k = per_kind.setdefault(kind, [0, 0.0, 0])
            k[0] += cells
            k[1] += sess.elapsed_ms(a, b)
            k[2] += 1
    sess.recycle()
    return per_kind


def _timed_session(plan, placement, dist, reps, warm=2):
    from paper_2505_06022_b200 import executor as E
    sess = E.Session(plan, placement, trace=True)
    sess.execute(upload=True)
    sess.synchronize()
    sess.recycle()
    for _ in range(warm):
        sess.execute(upload=False)
        sess.synchronize()
        sess.recycle()
    # traced stream replay (fallback only: host dispatch gaps inflate short launches)
    sess.execute(upload=False)
    sess.synchronize()
    log = [(k, c * reps, d, s, a, b) for k, c, d, s, a, b in sess.launch_log]
    per_kind = {}
    for kind, cells, _d, _s, a, b in log:
        k = per_kind.setdefault(kind, [0, 0.0, 0])
        k[0] += cells
        k[1] += sess.elapsed_ms(a, b) * reps
        k[2] += reps
    sess.recycle()
    per_kind = graph_launch_times(sess, reps) or per_kind
    graph = True
    try:
        sess.capture()
    except Exception:  # noqa: BLE001
        graph = False
        sess.synchronize()
        sess.recycle()
    dist.barrier()
    with ClockSampler(placement.devices[0]) as clocks:
        m0 = sess.mark()
        for _ in range(reps):
            if graph:
                sess.replay(1)
            else:
                sess.execute(upload=False)
        m1 = sess.mark()
        sess.synchronize()
    sess.clocks = clocks.summary()
    sess.clocks["replay"] = "cuda_graph" if graph else "stream"
    ms = max(sess.elapsed_ms(m0[d], m1[d]) for d in sess.devices)
    sess.recycle()
    return sess, dist.max(ms), per_kind, len(log) * reps


def energy_loop(sess, dist, ms_per_iter, seconds=1.0):
    """J per execute over >= ``seconds`` (NVML counter deltas).  The
    iteration count is agreed across ranks (every replay posts NCCL groups,
    so all ranks must run the same number)."""
    iters = int(dist.max(max(3, int(seconds * 1e3 / max(ms_per_iter, 1e-3)) + 1)))
    dist.barrier()
    try:
        e0 = sess.energy_mj()
    except Exception as exc:  # noqa: BLE001
        e0 = None
        err = str(exc)
    t0 = time.perf_counter()
    n = 0
    while n < iters:
        if getattr(sess, "graph", None):
            sess.replay(1)
        else:
            sess.execute(upload=False)
        n += 1
        if n % 4 == 0:
            sess.synchronize()
            sess.recycle()
    if e0 is None:
        sess.synchronize()
        sess.recycle()
        return {"error": err}
    sess.synchronize()
    sess.recycle()
    dt = time.perf_counter() - t0
    e1 = sess.energy_mj()
    joules = sum(e1[d] - e0[d] for d in e0) / 1000.0
    from paper_2505_06022_b200 import _native as N
    import ctypes
    cur, mx = ctypes.c_uint(), ctypes.c_uint()
    try:
        N.call("cq_nvml_sm_clock_mhz", sess.devices[0], ctypes.byref(cur), ctypes.byref(mx))
        clock = cur.value
    except Exception:  # noqa: BLE001
        clock = None
    return {"j_per_iter": joules / n, "watts": joules / dt, "iters": n, "seconds": dt,
            "sm_clock_mhz": clock}


def bench_kernels(args, dist, placement, peaks):
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import workloads as W
    world = dist.world
    sm_mhz = None
    out = {}
    fp32_peak = lambda mhz: 148 * 128 * 2 * mhz * 1e6 / 1e12  # noqa: E731

    # SAXPY: BASELINE config 0 exactly (2^24, one_to_one split into 4 chunks:
    # 4 plan nodes placed on the available GPUs) and a beyond-L2 point 2^28
    for n, label, nodes in ((1 << 24, "saxpy_2p24_4chunks", max(4, world)),
                            (1 << 28, "saxpy_2p28", world)):
        prog = W.saxpy_program(n, kind="float32")
        plan = cq.generate_commands(prog.graph(), nodes)
        sess, ms, kinds, launches = _timed_session(plan, placement, dist, reps=20)
        k = kinds.get("saxpy", [0, 1.0, 1])
        bracketed = dist.min(12 * k[0] / (k[1] / 1e3) / 1e9)
        value = 12 * n * 20 / (ms / 1e3) / 1e9
        # when the replayed graph holds nothing but the saxpy launches (no
        # copies), the region time / launch count is the average launch
        # duration back to back; event-record nodes around each launch add
        # ~2-3 us of node latency, which dominates 8-us launches
        only_saxpy = dist.min(1.0 if launches == k[2] else 0.0) == 1.0
        achieved = value / world if only_saxpy else bracketed
        out[label] = {"value": value, "unit": "GB/s", "scaling": "strong",
                      "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks[0]["hbm_gbs"],
                                   "frac": achieved / peaks[0]["hbm_gbs"],
                                   "achieved_event_bracketed": bracketed,
                                   "launch_timing": ("timed region / launches (graph of saxpy launches only)"
                                                     if only_saxpy else "timed CUDA-graph replay, event-bracketed")},
                      "chunks": nodes, "launches_per_pass": k[2] // 20,
                      "note": ("BASELINE config 0: 2^24 x fp32, 192 MiB per pass (> 126 MB L2; "
                               "back-to-back passes partly hit L2)") if n == 1 << 24 else "inputs > L2"}
        if args.energy and n == 1 << 28:
            e = energy_loop(sess, dist, ms / 20, 1.0)
            if e and "j_per_iter" in e:
                e["gb_per_joule"] = 12 * n / 1e9 / e["j_per_iter"]
            out[label]["energy"] = e
        sess.close()

    # wave variants: float64 (the reference's own element kind, 24 B/cell/step,
    # weak: 16384^2 per GPU) and strong scaling (global 16384^2 over N GPUs, fp32)
    for label, kind, rows, esize in (("wave_f64_weak", "float64", args.size * world, 24),
                                     ("wave_f32_strong", "float32", args.size, 12)):
        steps = 20
        z = np.zeros((1, 1))
        from paper_2505_06022_b200.model import Buffer, BufferInit
        from paper_2505_06022_b200.region import Box
        ext = Box.from_shape((rows, args.size))
        bufs = {"u": Buffer("u", ext, kind, BufferInit.constant(0.5)),
                "up": Buffer("up", ext, kind, BufferInit.constant(0.25))}
        tasks = [W.wave_task(s, rows, args.size, C) for s in range(steps)]
        g = cq.TaskGraph(bufs)
        for t in tasks:
            g.submit(t)
        del z
        plan = cq.generate_commands(g, world)
        sess, ms, kinds, _ = _timed_session(plan, placement, dist, reps=3, warm=1)
        fk = max((k for k in kinds if k.startswith("wave5")), key=lambda k: kinds[k][0], default="wave5")
        # algorithmic bytes per cell per launch: fused = read X(t), X(t-1) and
        # write two levels (4 elements), one-step = 3 elements
        kb = esize // 3 * 4 if fk != "wave5" else esize
        wk = kinds.get(fk, [0, 1.0, 1])
        value = esize * rows * args.size * steps * 3 / (ms / 1e3) / 1e9
        out[label] = {"value": value, "unit": "GB/s", "scaling": "weak" if "weak" in label else "strong",
                      "bytes_per_cell": esize, "time_steps": steps, "ms_per_time_step": ms / 3 / steps,
                      "kernel": fk, "kernel_gbs_min_rank": dist.min(kb * wk[0] / (wk[1] / 1e3) / 1e9),
                      "clocks": sess.clocks}
        sess.close()

    # N-body: 262144 bodies, 'all' mapper all-gather each step
    nb = args.nbody
    prog = W.nbody_program(nb, steps=3)
    plan = cq.generate_commands(prog.graph(), world)
    sess, ms, kinds, _ = _timed_session(plan, placement, dist, reps=3, warm=1)
    clocks = sess.clocks
    kick = kinds.get("nbody.kick", [0, 1.0, 1])
    inter = nb * nb * 3 * 3
    gflops = 20 * inter / (ms / 1e3) / 1e9
    if world == 1:
        kick_gflops = dist.min(20 * (kick[0] // 4) * nb / (kick[1] / 1e3) / 1e9)
        kick_timing = "kick launches' CUDA-event time"
    else:
        # the kick runs as concurrent launches (held j columns / arriving ones,
        # executor.exec_kick): summed launch times would over-count, so the
        # per-GPU rate comes from the whole step's device time (kick, drift and
        # the overlapped all-gather; a lower bound on the kick's own rate)
        kick_gflops = gflops / world
        kick_timing = "whole step's device time per GPU (kick launches overlap the all-gather)"
    energy = energy_loop(sess, dist, ms / 3, 1.0) if args.energy else None
    clk = clocks.get("sm_mhz") or (energy or {}).get("sm_clock_mhz")
    out["nbody_262144"] = {"value": gflops, "unit": "GFLOP/s", "scaling": "strong",
                           "ms_per_step": ms / 9, "flop_per_interaction": 20,
                           "roofline": {"bound": "fp32", "achieved": kick_gflops,
                                        "peak": fp32_peak(1965) * 1e3, "unit": "GFLOP/s",
                                        "frac": kick_gflops / 1e3 / fp32_peak(1965),
                                        "frac_at_observed_clock":
                                            (kick_gflops / 1e3 / fp32_peak(clk)) if clk else None,
                                        "peak_definition": "148 SM x 128 FP32 lanes x 2 flop x 1965 MHz",
                                        "timing": kick_timing},
                           "clocks": clocks, "energy": energy}
    sess.close()

    # sgemm 16384^3 (slice mappers): 3xTF32 on tcgen05 and the FFMA baseline
    tf32_ceiling = peaks[0].get("bf16_tflops", 1649.2) / 2 / 3
    for variant in args.sgemm_variants:
        m = args.sgemm
        a = np.empty((m, m), np.float32)
        b = np.empty((m, m), np.float32)
        rng = np.random.default_rng(5)
        a[...] = rng.uniform(-1, 1, (m, m)).astype(np.float32)
        b[...] = rng.uniform(-1, 1, (m, m)).astype(np.float32)
        prog = W.sgemm_program(m, m, m, variant=variant, a=a, b=b)
        plan = cq.generate_commands(prog.graph(), world)
        try:
            sess, ms, kinds, _ = _timed_session(plan, placement, dist, reps=3, warm=1)
        except Exception as exc:  # noqa: BLE001
            out[f"sgemm_{variant}"] = {"error": str(exc)}
            continue
        tflops = 2 * m ** 3 * 3 / (ms / 1e3) / 1e12
        # per-GPU kernel rate from the traced launch (includes the hi/lo split pass)
        sk = kinds.get("sgemm", [0, 1.0, 1])
        kern_tflops = dist.min(2 * sk[0] * m / (sk[1] / 1e3) / 1e12)
        entry = {"value": tflops * 1e3, "unit": "GFLOP/s (useful 2MNK)", "scaling": "strong",
                 "per_gpu_kernel_tflops": kern_tflops,
                 "frac_of_fp32_simt_peak_at_max_clock": kern_tflops / fp32_peak(1965),
                 "clocks": sess.clocks}
        if variant == "3xtf32":
            sustained = peaks[0].get("bf16_tflops_sustained", 1377.2) / 2 / 3
            entry["roofline"] = {"bound": "tensor", "achieved": kern_tflops, "unit": "TFLOP/s",
                                 "peak": tf32_ceiling, "frac": kern_tflops / tf32_ceiling,
                                 "peak_sustained": sustained, "frac_sustained": kern_tflops / sustained,
                                 "peak_definition": "measured bf16 dense (burst | sustained) / 2 (TF32) "
                                                    "/ 3 (products)"}
        if args.energy and variant == "3xtf32":
            e = energy_loop(sess, dist, ms / 3, 1.0)
            if e and "j_per_iter" in e:
                e["tflop_per_joule"] = 2 * m ** 3 / 1e12 / e["j_per_iter"]
            entry["energy"] = e
        out[f"sgemm_{variant}_{m}"] = entry
        sess.close()
    return out


# ------------------------------------------------------------- CPU baselines

def _all_host_threads():
    """torchrun exports OMP_NUM_THREADS=1; the CPU arms use every core
    (must be set before the OpenMP runtime of the oracle library loads)."""
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())


def cpu_wave_baseline(seconds=12.0, size=SIZE):
    """The CPU port of the wave step (oracle/cq_oracle.c, OpenMP over all
    host threads) on the same 16384^2 fp32 grid, bounded to ~``seconds``."""
    _all_host_threads()
    from oracle import native as onat
    u = np.random.default_rng(2).uniform(0, 1, (size, size)).astype(np.float32)
    up = u.copy()
    onat.wave_step(u, up, C, out=up)  # warm
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        if n % 2 == 0:
            onat.wave_step(u, up, C, out=up)
        else:
            onat.wave_step(up, u, C, out=u)
        n += 1
    dt = time.perf_counter() - t0
    return {"value": 12 * size * size * n / dt / 1e9, "unit": "GB/s", "cores": os.cpu_count(),
            "kind": "port", "sample": f"{n} wave steps of {size}x{size} fp32 "
                                      f"(oracle/cq_oracle.c, OpenMP, {os.cpu_count()} threads)"}


def cpu_kernel_baselines(args, seconds=4.0):
    """SURVEY §8d's CPU-side column for SAXPY, N-body and matmul: the C port
    (oracle/cq_oracle.c, OpenMP over every host thread) on bounded samples
    of the same workloads, ~``seconds`` each."""
    _all_host_threads()
    from oracle import native as onat
    from paper_2505_06022_b200 import workloads as W
    cores = os.cpu_count()
    out = {}

    def loop(fn):
        fn()  # warm
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < seconds:
            fn()
            n += 1
        return n, time.perf_counter() - t0

    n = 1 << 24
    x, y = W.saxpy_inputs(n, "float32", seed=0)
    reps, dt = loop(lambda: onat.saxpy(2.0, x, y))
    out["saxpy_2p24_4chunks"] = {"value": 12 * n * reps / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
                                 "sample": f"{reps} fp32 SAXPY passes over 2^24 elements (12 B/element)"}
    nb = args.nbody
    pos, _vel = W.nbody_inputs(nb)
    ni = 64
    reps, dt = loop(lambda: onat.nbody_accel(pos, 0, ni, 1e-2))
    out["nbody_262144"] = {"value": 20 * ni * nb * reps / dt / 1e9, "unit": "GFLOP/s", "cores": cores,
                           "kind": "port",
                           "sample": f"{reps} x {ni} i-bodies x all {nb} j (float64 accumulation, fixed j order; "
                                     "20 flop/interaction)"}
    m = args.sgemm
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (8, m)).astype(np.float32)
    b = rng.uniform(-1, 1, (m, m)).astype(np.float32)
    rows = np.arange(8)
    reps, dt = loop(lambda: onat.sgemm_rows(a, b, rows, with_abs=False))
    out["sgemm"] = {"value": 2 * 8 * m * m * reps / dt / 1e9, "unit": "GFLOP/s (useful 2MNK)", "cores": cores,
                    "kind": "port", "sample": f"{reps} x 8 rows of C = A B at K = N = {m} (float64 accumulation, "
                                              "fixed k order)"}
    return out


def cpu_baselines_in_subprocess(args, kernels=True):
    """The CPU legs in a fresh process: this one has torch (and its OpenMP
    runtime, sized by torchrun's OMP_NUM_THREADS=1 or torch's own setting)
    loaded, which would pin the C port to fewer threads than the host has."""
    env = dict(os.environ, OMP_NUM_THREADS=str(os.cpu_count()))
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-only", "--size", str(args.size),
           "--nbody", str(args.nbody), "--sgemm", str(args.sgemm)] + ([] if kernels else ["--no-kernels"])
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else {"wave": {"error": r.stderr[-300:]}}
    except (OSError, subprocess.TimeoutExpired, ValueError) as exc:
        return {"wave": {"error": str(exc)[:300]}}


def reference_arm(args, dist):
    """--impl reference: the reference's CPU implementation of the path on the
    host cores.  The reference is pure Python (clusterq, ~50 us per cell) and
    does not travel to the GPU box, so this times its C restatement
    (oracle/cq_oracle.c, OpenMP over every host thread) on the b200 arm's
    workload: each bench step is one full ``--wave-steps`` simulation of one
    GPU's 16384 x 16384 fp32 slab from the same Gaussian pulse.  At N > 1 the
    whole job is N such slabs; the CPU's rate does not depend on how many, so
    one slab per step is the bounded sample (rank 0 alone runs)."""
    if dist.rank != 0:
        return None
    _all_host_threads()
    from oracle import native as onat
    size, nsteps = args.size, args.wave_steps
    u0 = pulse_field(size, size)

    def simulate():
        # ping-pong as workloads.wave_program: even steps write up, odd steps u
        u, up = u0.copy(), u0.copy()
        for s in range(nsteps):
            if s % 2 == 0:
                onat.wave_step(u, up, C, out=up)
            else:
                onat.wave_step(up, u, C, out=u)

    for _ in range(args.warmup):
        simulate()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        simulate()
    dt = time.perf_counter() - t0
    val = 12 * size * size * nsteps * args.steps / dt / 1e9
    sample = (f"{args.steps} x {nsteps}-step simulations of one {size}x{size} fp32 slab (Gaussian pulse), "
              f"oracle/cq_oracle.c OpenMP {os.cpu_count()} threads"
              + (f"; the {args.gpus}-GPU job is {args.gpus} such slabs" if args.gpus > 1 else ""))
    return {
        "metric": METRIC, "impl": "reference", "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": headline_config(size, args.gpus, nsteps),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def clock_sweep(args, dist, placement):
    """SYnergy sweep (BASELINE config 4): J and seconds per iteration of the
    100-step wave simulation and of 3 N-body steps at three SM clocks (max,
    ~75%, ~50% of the supported list), the reference time model's beta fitted
    per kernel, and the reference selection rule per target over the measured
    points.  Locking clocks changes shared hardware state, so it runs only
    with CQ_ALLOW_CLOCK_LOCK=1 (libcq refuses otherwise) and at N = 1."""
    if os.environ.get("CQ_ALLOW_CLOCK_LOCK") != "1":
        return ("not run: SM clock locking is disabled on this shared pool (cq_nvml_lock_sm_clock "
                "requires CQ_ALLOW_CLOCK_LOCK=1); J/iteration reported at the running clock")
    if dist.world != 1:
        return "not run: the sweep is a 1-GPU measurement"
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import executor as E, synergy as S, workloads as W
    from paper_2505_06022_b200.energy import EnergyTarget
    dev = placement.devices[0]
    clocks = S.sweep_clocks(S.supported_sm_clocks(dev))
    out = {"clocks_mhz": clocks}
    u0, up0 = wave_inputs(args.size, args.size, (0, args.size))
    programs = {"wave5_100_steps": W.wave_program(args.size, args.size, steps=args.wave_steps, c=C, u0=u0, up0=up0),
                "nbody_3_steps": W.nbody_program(args.nbody, steps=3)}
    for name, prog in programs.items():
        sess = E.Session(cq.generate_commands(prog.graph(), 1), placement, trace=False)
        sess.execute(upload=True)
        sess.synchronize()
        sess.recycle()
        sess.capture()
        mk = S.sweep(name, lambda: sess.replay(1), dev, clocks, seconds=SWEEP_SECONDS, sync=sess.synchronize)
        entry = {"points": {str(m): {"s_per_iter": t, "j_per_iter": j} for m, (t, j) in sorted(mk.points.items())}}
        if len(mk.points) > 1:
            entry["beta"] = float(S.fit_beta(mk))
            entry["selected_mhz"] = {t.value: S.select_measured(mk, t) for t in EnergyTarget}
        out[name] = entry
        sess.close()
    return out


def headline_line(args, world, wave, cpu, kernels, sweep):
    """The b200 arm's JSON line; metric, unit, higher_is_better and config
    are the reference arm's (``reference_arm``) byte for byte."""
    return {
        "metric": METRIC, "impl": "b200", "value": wave["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wave["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": headline_config(args.size, world, args.wave_steps),
        "run": {"plan_s": wave["plan_s"], "replay": wave["replay"], "execution": wave["execution"],
                "kernels_note": "per-kernel GB/s | GFLOP/s and % roofline of the other BASELINE workloads "
                                "are under 'kernels'"},
        "e2e": wave["e2e"], "roofline": wave["roofline"], "cpu_baseline": cpu,
        "clocks": wave["clocks"], "gpu_launches": wave["gpu_launches"],
        "energy": {"wave5": wave["energy"], "clock_sweep": sweep},
        "kernels": kernels,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", type=int, default=SIZE)
    ap.add_argument("--wave-steps", type=int, default=WAVE_STEPS)
    ap.add_argument("--nbody", type=int, default=262144)
    ap.add_argument("--sgemm", type=int, default=16384)
    ap.add_argument("--sgemm-variants", default="3xtf32,ffma")
    ap.add_argument("--no-kernels", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-energy", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="replay via per-command stream dispatch")
    ap.add_argument("--cpu-only", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.cpu_only:   # the CPU legs of the b200 arm (cpu_baselines_in_subprocess)
        out = {"wave": cpu_wave_baseline(size=args.size)}
        if not args.no_kernels:
            out.update(cpu_kernel_baselines(args))
        print(json.dumps(out))
        return 0
    args.sgemm_variants = [v for v in args.sgemm_variants.split(",") if v]
    args.energy = not args.no_energy

    if args.impl == "reference":
        # rank 0 alone runs the CPU reference arm; other ranks exit at once
        if _env_int("RANK", 0) != 0:
            return 0

        class _Rank0:
            rank = 0
        print(json.dumps(reference_arm(args, _Rank0())))
        return 0

    dist = Dist(args.gpus)
    from paper_2505_06022_b200 import executor as E
    if dist.world > 1:
        placement = E.init_distributed(dist.rank, dist.world, dist.local_rank)
    else:
        placement = E.Placement(1, 0, (0,))
    peaks = measured_peaks()
    wave = bench_wave(args, dist, placement, peaks)
    kernels = None if args.no_kernels else bench_kernels(args, dist, placement, peaks)
    cpu = None
    if dist.world == 1 and dist.rank == 0 and not args.no_cpu:
        base = cpu_baselines_in_subprocess(args, kernels is not None)
        cpu = base.pop("wave", None)
        for key, entry in (kernels or {}).items():
            for name, b in base.items():
                if key.startswith(name) and isinstance(entry, dict):
                    entry["cpu_baseline"] = b
    if dist.rank == 0:
        sweep = clock_sweep(args, dist, placement) if args.energy else None
        line = headline_line(args, dist.world, wave, cpu, kernels, sweep)
        print(json.dumps(line))
    if dist.world > 1:
        E.shutdown_distributed()
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
