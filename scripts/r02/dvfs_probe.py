"""Read-only DVFS probe (changes no clock setting).  The B200's own power
management moves the SM clock under a sustained kernel (the wave pass hits
the 1 kW cap and drops from 1965 MHz to ~1650 within ~0.2 s); this records
time per iteration against the SM clock the GPU chose, and the NVML energy
counter, so the SYnergy time model's beta (energy.py:74-78) can be fitted
from hardware points without locking clocks (the pool forbids it).

A sampler *process* (own GIL) reads SM clock, power and the energy counter
every ~1 ms; the main process replays a captured graph back to back, one
synchronize per iteration, in bursts separated by idle gaps (each burst
starts at the idle clock).  Output: JSON on stdout."""
import json
import multiprocessing as mp
import sys
import time

sys.path.insert(0, ".")


def sampler(conn, stop):
    import ctypes
    from paper_2505_06022_b200 import _native as N, synergy as S
    out = []
    pw = ctypes.c_uint()
    while not stop.is_set():
        t = time.perf_counter()
        N.call("cq_nvml_power_mw", 0, ctypes.byref(pw))
        out.append((t, S.sm_clock(0)[0], pw.value, S.energy_mj(0)))
        time.sleep(0.001)
    conn.send(out)


def probe(name, prog, bursts, seconds, idle):
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import executor as E
    sess = E.Session(cq.generate_commands(prog.graph(), 1), E.Placement(1, 0, (0,)), trace=False)
    sess.execute(upload=True)
    sess.synchronize()
    sess.recycle()
    sess.capture()
    ctx = mp.get_context("spawn")
    rx, tx = ctx.Pipe(duplex=False)
    stop = ctx.Event()
    p = ctx.Process(target=sampler, args=(tx, stop))
    p.start()
    iters = []
    for _ in range(bursts):
        time.sleep(idle)
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            a = time.perf_counter()
            sess.replay(1)
            sess.synchronize()
            iters.append((a, time.perf_counter()))
    time.sleep(0.3)
    stop.set()
    samples = rx.recv()
    p.join()
    sess.close()
    return {"name": name, "iters": iters, "samples": samples}


def main():
    from paper_2505_06022_b200 import workloads as W
    n = 16384
    u0 = W.wave_pulse(n, n, "float32")
    res = [probe("wave5_100_steps", W.wave_program(n, n, steps=100, c=0.25, u0=u0, up0=u0), 4, 2.0, 2.5),
           probe("nbody_3_steps", W.nbody_program(262144, steps=3), 1, 3.0, 1.0)]
    json.dump(res, sys.stdout)


if __name__ == "__main__":
    main()
