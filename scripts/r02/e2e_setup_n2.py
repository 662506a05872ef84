"""e2e at N ranks: cost of Session setup / close (IPC peer-halo opening at
N > 1) against run_batch per-simulation time for 5 and 15 jobs per call.

    torchrun --nproc-per-node 2 scripts/r02/e2e_setup_n2.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.region import Box  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
S = 16384
H, Wd = S * world, S
lo, hi = rank * S, (rank + 1) * S
u0 = E.pinned_empty((H, Wd), np.float32, Box((max(lo - 1, 0), 0), (min(hi + 1, H), Wd)))
u0[max(lo - 1, 0):min(hi + 1, H)] = 0.5
prog = W.wave_program(H, Wd, steps=100, kind="float32", c=0.25, u0=u0, up0=u0)
plan = cq.generate_commands(prog.graph(), world)
pl = E.init_distributed(rank, world, rank)
outs = [{"u": E.pinned_empty((H, Wd), np.float32, Box((lo, 0), (hi, Wd))),
         "up": E.pinned_empty((H, Wd), np.float32, Box((lo, 0), (hi, Wd)))} for _ in range(3)]


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


E.run_batch(plan, [(None, outs[k % 3]) for k in range(6)], gather="local", depth=3, placement=pl)
for rep in range(3):
    dist.barrier()
    t0 = time.perf_counter()
    s = E.Session(plan, pl, trace=False)
    t1 = time.perf_counter()
    s.close()
    t2 = time.perf_counter()
    mk, cl = tmax(t1 - t0), tmax(t2 - t1)
    if rank == 0:
        print(f"session create {mk * 1e3:.1f} ms, close {cl * 1e3:.1f} ms", flush=True)
for jobs in (5, 15, 5, 15):
    dist.barrier()
    t0 = time.perf_counter()
    E.run_batch(plan, [(None, outs[k % 3]) for k in range(jobs)], gather="local", depth=3, placement=pl)
    dt = tmax(time.perf_counter() - t0)
    if rank == 0:
        print(f"run_batch {jobs} jobs: {dt * 1e3 / jobs:.1f} ms/sim ({dt * 1e3:.0f} ms)", flush=True)
dist.destroy_process_group()
