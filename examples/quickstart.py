"""Quickstart: the reference's clusterq API on B200s.

    python examples/quickstart.py            # one process, all visible GPUs
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 examples/quickstart.py   # one rank per GPU

Builds the bundled SAXPY scenario and a 2-D wave simulation with the
reference's own front end (Buffer / Accessor / Task / TaskGraph.submit, range
mappers), plans them with generate_commands (identical Plans to clusterq) and
runs them with run(plan) on the GPUs; prints the SYnergy energy report of the
measured trace.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2505_06022_b200 as clusterq  # noqa: E402  (was: import clusterq)
from paper_2505_06022_b200 import executor  # noqa: E402


def saxpy(n, nodes):
    ext = clusterq.Box.from_shape((n,))
    bufs = {"x": clusterq.Buffer("x", ext, "float32", clusterq.BufferInit.iota()),
            "y": clusterq.Buffer("y", ext, "float32", clusterq.BufferInit.constant(1.0)),
            "z": clusterq.Buffer("z", ext, "float32", clusterq.BufferInit.zeros())}
    g = clusterq.TaskGraph(bufs)
    body = {"z": clusterq.parse_kernel("alpha * x[i] + y[i]", {"x": 1, "y": 1}, {"alpha"}, 1)}
    g.submit(clusterq.Task("saxpy", ext, [clusterq.Accessor("x", clusterq.AccessMode.READ),
                                          clusterq.Accessor("y", clusterq.AccessMode.READ),
                                          clusterq.Accessor("z", clusterq.AccessMode.WRITE)],
                           body, params={"alpha": 2.0}))
    plan = clusterq.generate_commands(g, nodes)
    res = clusterq.run(plan)
    if res.buffers:
        assert np.array_equal(res.buffers["z"], 2.0 * np.arange(n, dtype=np.float32) + 1.0)
    return plan, res


def wave(h, w, steps, nodes):
    from paper_2505_06022_b200 import workloads as W
    prog = W.wave_program(h, w, steps=steps, kind="float32", c=0.25)
    plan = clusterq.generate_commands(prog.graph(), nodes)
    return plan, clusterq.run(plan, energy=True)


def main():
    if "RANK" in os.environ:   # torchrun: one process per GPU, NCCL between ranks
        import torch
        import torch.distributed as dist
        rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        executor.init_distributed(rank, world, local)
        nodes = world
    else:
        nodes, rank = 4, 0
    plan, res = saxpy(1 << 24, nodes)
    plan, res = wave(4096, 4096, 96, nodes)
    if rank == 0:
        report = clusterq.account_energy(res.trace, plan.devices, res.makespan)
        print(f"wave 4096^2 x 96 steps on {nodes} nodes: makespan {float(res.makespan) * 1e3:.2f} ms, "
              f"model energy {float(report.total_device_energy):.2f} J, measured {res.measured}")
    if "RANK" in os.environ:
        executor.shutdown_distributed()


if __name__ == "__main__":
    main()
