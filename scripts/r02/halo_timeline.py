"""Per-pass device timeline of the temporally blocked wave at N ranks (one
GPU each, the bench's weak-scaled 16384^2-per-GPU x 100 steps): for every
pass the interior launch, the neighbour-edge launches and the KL-row halo
exchange (start / end in ms from the replay's first launch), read from
event-record nodes of a timed CUDA-graph replay.

    torchrun --nproc-per-node N scripts/r02/halo_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import bench  # noqa: E402
import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
pl = E.init_distributed(rank, world, local)
S = 16384
H = S * world
lo, hi = rank * S, (rank + 1) * S
u0, up0 = bench.wave_inputs(H, S, (lo, hi))
plan = cq.generate_commands(W.wave_program(H, S, steps=100, kind="float32", c=0.25, u0=u0, up0=up0).graph(), world)

halo = []
orig = E.Session.exec_fused


def exec_fused(self, *a, **k):
    orig(self, *a, **k)
    if self.want_trace:
        halo.append([(m[3], m[4]) for m in self._halo_marks])


E.Session.exec_fused = exec_fused
s = E.Session(plan, pl, trace=True)
s.execute(upload=True)
s.synchronize()
s.recycle()
halo.clear()
s.capture(timed=True)
for _ in range(3):
    s.replay(1)
    s.synchronize()
log = s.graph_log
t0 = log[0][4]
rel = lambda ev: s.elapsed_ms(t0, ev)  # noqa: E731
lines = [f"rank {rank}/{world}: {len(log)} launches, replay {rel(log[-1][5]):.3f} ms"]
for kind, cells, _d, stream, a, b in log:
    lines.append(f"  {kind:13s} stream {stream} rows {cells // S:6d} {rel(a):8.3f} - {rel(b):8.3f} ms")
for i, h in enumerate(halo):
    if h:
        lines.append(f"  halo pass {i:2d}: {min(rel(a) for a, _ in h):8.3f} - {max(rel(b) for _, b in h):8.3f} ms")
out = [None] * world
dist.all_gather_object(out, "\n".join(lines))
if rank == 0:
    print("\n\n".join(out), flush=True)
s.close()
E.shutdown_distributed()
dist.destroy_process_group()
