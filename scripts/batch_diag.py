"""Host-side timeline of run_batch across ranks (torchrun, one GPU per rank):
per job, the wall time spent inside Session.execute / issue_results /
finish_results, and the whole batch, for a few depths and job counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402
from paper_2505_06022_b200.region import Box  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pl = E.init_distributed(rank, world, local)
    size = int(os.environ.get("DIAG_SIZE", "16384"))
    H, Wd = size * world, size
    lo, hi = rank * size, (rank + 1) * size
    rows = Box((max(lo - 1, 0), 0), (min(hi + 1, H), Wd))
    u0 = E.pinned_empty((H, Wd), np.float32, rows)
    up0 = E.pinned_empty((H, Wd), np.float32, rows)
    u0[rows.mins[0]:rows.maxs[0]] = 0.5
    up0[rows.mins[0]:rows.maxs[0]] = 0.5
    prog = W.wave_program(H, Wd, steps=100, kind="float32", c=0.25, u0=u0, up0=up0)
    plan = cq.generate_commands(prog.graph(), world)
    out_box = Box((lo, 0), (hi, Wd))
    log = []
    for name in ("execute", "issue_results", "finish_results", "recycle", "__init__", "close"):
        orig = getattr(E.Session, name)

        def wrap(self, *a, _o=orig, _n=name, **k):
            t = time.perf_counter()
            r = _o(self, *a, **k)
            log.append((_n, id(self) % 1000, t, time.perf_counter()))
            return r
        setattr(E.Session, name, wrap)
    gather = "local" if world > 1 else "root"
    for depth, jobs in ((3, 3), (3, 6), (1, 3)):
        outs = [{"u": E.pinned_empty((H, Wd), np.float32, out_box),
                 "up": E.pinned_empty((H, Wd), np.float32, out_box)} for _ in range(depth)]
        E.run_batch(plan, [(None, outs[k % depth]) for k in range(depth)], gather=gather, depth=depth)
        dist.barrier()
        log.clear()
        t0 = time.perf_counter()
        E.run_batch(plan, [(None, outs[k % depth]) for k in range(jobs)], gather=gather, depth=depth)
        total = time.perf_counter() - t0
        lines = [f"rank {rank} depth {depth} jobs {jobs}: {total * 1e3:.1f} ms total, {total / jobs * 1e3:.1f} ms/job"]
        for n, sid, a, b in log:
            lines.append(f"   {n:15s} s{sid:03d} {1e3 * (a - t0):8.1f} -> {1e3 * (b - t0):8.1f} ms ({1e3 * (b - a):7.1f})")
        for r in range(world):
            if r == rank:
                print("\n".join(lines), flush=True)
            dist.barrier()
    E.shutdown_distributed()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
