"""Summarise dvfs_probe.py output: time per iteration against the SM clock
the GPU's power management chose (no clock was set), joules per iteration
from the NVML energy counter's steps, and the SYnergy time model's beta
(energy.py:74-78) fitted from those observed points with synergy.fit_beta.
Usage: python scripts/r02/dvfs_summary.py probe.json"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2505_06022_b200 import synergy as S  # noqa: E402
from paper_2505_06022_b200.energy import EnergyTarget  # noqa: E402


def clock_bins(r):
    """{state: [(mhz, s/iter)]}: 'max' = iterations at the idle/max clock,
    'capped' = iterations after the power limiter pulled the clock down."""
    s, it = np.array(r["samples"]), np.array(r["iters"])
    rows = []
    for a, b in it:
        m = (s[:, 0] >= a) & (s[:, 0] <= b)
        if m.sum():
            rows.append((float(np.median(s[m, 1])), b - a))
    return np.array(rows)


def energy_windows(r):
    """(median clock, W, J/iter) over the counter-step windows fully covered
    by iterations."""
    s, it = np.array(r["samples"]), np.array(r["iters"])
    idx = [i for i in range(1, len(s)) if s[i, 3] != s[i - 1, 3]]
    out = []
    for a, b in zip(idx[:-1], idx[1:]):
        t0, t1 = s[a, 0], s[b, 0]
        busy = np.sum(np.clip(np.minimum(it[:, 1], t1) - np.maximum(it[:, 0], t0), 0, None))
        inside = (it[:, 0] >= t0) & (it[:, 1] <= t1)
        if busy / (t1 - t0) > 0.95 and inside.sum():
            w = (s[b, 3] - s[a, 3]) / 1000.0 / (t1 - t0)
            out.append((float(np.median(s[a:b + 1, 1])), w, w * float(np.mean(it[inside, 1] - it[inside, 0]))))
    return out


def main(path):
    res = json.load(open(path))
    for r in res:
        rows = clock_bins(r)
        top = rows[:, 0].max()
        hi, lo = rows[rows[:, 0] >= top - 1], rows[rows[:, 0] < top - 1]
        ew = energy_windows(r)
        print(f"{r['name']}: {len(r['iters'])} iterations, {len(r['samples'])} NVML samples")
        pts = {}
        for label, part in (("max", hi), ("power-capped", lo)):
            if not len(part):
                print(f"  {label}: no iterations")
                continue
            mhz = int(round(float(np.median(part[:, 0]))))
            t = float(np.median(part[:, 1]))
            js = [j for c, _, j in ew if (c >= top - 1) == (label == "max")]
            ws = [w for c, w, _ in ew if (c >= top - 1) == (label == "max")]
            j = float(np.median(js)) if js else float("nan")
            print(f"  {label:12s}: SM {mhz} MHz (observed, median; range {part[:, 0].min():.0f}-{part[:, 0].max():.0f}), "
                  f"{len(part)} iterations, {1e3 * t:.2f} ms/iter, {j:.2f} J/iter "
                  f"({np.median(ws) if ws else float('nan'):.0f} W, {len(js)} counter windows)")
            if js:
                pts[mhz] = (t, j)
        if len(pts) >= 2:
            mk = S.MeasuredKernel(r["name"], pts)
            print(f"  beta (reference time model, fitted on the observed points) = {float(S.fit_beta(mk)):.3f}")
            print("  reference selection over the observed points: " +
                  ", ".join(f"{t.value} -> {S.select_measured(mk, t)} MHz" for t in EnergyTarget))


if __name__ == "__main__":
    main(sys.argv[1])
