"""Multi-rank correctness check (one process per GPU, NCCL between ranks).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P scripts/mgpu_check.py

Every rank builds the same programs (Celerity's model); rank 0 gathers and
compares against the CPU oracle.  Exit code 0 iff every check passes."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import executor as E  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pl = E.init_distributed(rank, world, local)
    failures = []

    def check(name, ok):
        if rank == 0:
            print(f"{'PASS' if ok else 'FAIL'} {name}", flush=True)
            if not ok:
                failures.append(name)

    from oracle import dsl
    from oracle import native as onat

    # wave ping-pong, nodes = world and 2*world - 1 (uneven slabs)
    # (temporally blocked when the chain is >= 8 steps: KL-row halo exchange
    # between ranks; CQ_WAVE_FUSE=0 runs the per-step plan)
    h, w = 515, 384
    u0 = np.random.default_rng(2).uniform(0, 1, (h, w)).astype(np.float32)
    up0 = np.random.default_rng(3).uniform(0, 1, (h, w)).astype(np.float32)
    for steps, fuse in ((9, "1"), (9, "0"), (22, "1")):
        os.environ["CQ_WAVE_FUSE"] = fuse
        for nodes in sorted({world, max(1, 2 * world - 1)}):
            prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=up0)
            res = E.run(cq.generate_commands(prog.graph(), nodes), placement=pl)
            if rank == 0:
                u, up = onat.wave_run(u0, up0, steps, 0.25)
                check(f"wave {h}x{w}x{steps} nodes={nodes} fuse={fuse}",
                      dsl.same_bits(res.buffers["u"], u) and dsl.same_bits(res.buffers["up"], up))
    os.environ.pop("CQ_WAVE_FUSE")

    # float64 (the reference's kind) chain, temporally blocked across ranks
    d0 = np.random.default_rng(4).uniform(0, 1, (h, w))
    prog = W.wave_program(h, w, steps=18, kind="float64", c=0.3, u0=d0, up0=d0)
    res = E.run(cq.generate_commands(prog.graph(), world), placement=pl)
    if rank == 0:
        u, up = onat.wave_run(d0, d0, 18, 0.3)
        check(f"wave float64 {h}x{w}x18 nodes={world}",
              dsl.same_bits(res.buffers["u"], u) and dsl.same_bits(res.buffers["up"], up))

    # run_batch across ranks: simulations in flight, each rank reads back its
    # rows -- halo rows over NCCL (run_batch's default), then with the
    # peer-memory path forced (CQ_WAVE_P2P=1) unless the caller disabled it
    prog = W.wave_program(h, w, steps=12, kind="float32", u0=u0, up0=up0)
    plan = cq.generate_commands(prog.graph(), world)
    mine = next(c for c in plan.commands if type(c).__name__ == "ExecuteCommand" and c.node == rank)
    lo, hi = mine.chunk.box.mins[0], mine.chunk.box.maxs[0]
    env0 = os.environ.get("CQ_WAVE_P2P")
    for mode in ("nccl", "peer"):
        if mode == "peer":
            if env0 == "0":
                continue
            os.environ["CQ_WAVE_P2P"] = "1"
        before = E.STATS["peer_blocks"]
        jobs = [(None, None), ({"u": up0, "up": u0}, None), (None, None)]
        batch = E.run_batch(plan, jobs, gather="local")
        used = E.STATS["peer_blocks"] - before
        ok = True
        for (inp, _o), r in zip(jobs, batch):
            a, b = (u0, up0) if inp is None else (up0, u0)
            u, up = onat.wave_run(a, b, 12, 0.25)
            ok = ok and dsl.same_bits(r["u"][lo:hi], u[lo:hi]) and dsl.same_bits(r["up"][lo:hi], up[lo:hi])
        if world > 1 and env0 is None:
            ok = ok and ((used > 0) == (mode == "peer"))
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        check(f"run_batch 3 jobs nodes={world}, halo rows via {mode} ({used} peer blocks; every rank's own rows)",
              bool(flag.item()))
    if env0 is None:
        os.environ.pop("CQ_WAVE_P2P", None)
    else:
        os.environ["CQ_WAVE_P2P"] = env0

    # SAXPY, BASELINE config 1 shape scaled
    n = (1 << 22) + 5
    x, y = W.saxpy_inputs(n, "float32", seed=0)
    prog = W.saxpy_program(n, kind="float32", x=x, y=y)
    res = E.run(cq.generate_commands(prog.graph(), world), placement=pl)
    if rank == 0:
        check(f"saxpy {n}", dsl.same_bits(res.buffers["z"], onat.saxpy(2.0, x, y)))

    # N-body: all-gather of positions each step; bit-identical to 1 GPU
    nb = 4096
    pos, vel = W.nbody_inputs(nb)
    prog = W.nbody_program(nb, steps=2, pos=pos, vel=vel)
    before = E.STATS["allgather"]
    res = E.run(cq.generate_commands(prog.graph(), world), placement=pl)
    # the second step's 'all' exchange is one in-place ncclAllGather
    check(f"nbody {nb} x2 steps: the 'all' exchange ran as ncclAllGather "
          f"({E.STATS['allgather'] - before} call)", E.STATS["allgather"] - before == 1)
    if rank == 0:
        # the j order is fixed independently of the GPU count, so the
        # distributed result equals a 1-GPU run of the same program bit for bit
        single = E.run(cq.generate_commands(prog.graph(), 1), placement=E.Placement(1, 0, (local,)))
        ok = dsl.same_bits(res.buffers["P"], single.buffers["P"]) and \
            dsl.same_bits(res.buffers["V"], single.buffers["V"])
        acc = onat.nbody_accel(pos, 0, nb, 1e-2)
        # one kick from rest: V = dt * a within the SURVEY §8d tolerance
        prog1 = W.nbody_program(nb, steps=1, pos=pos, vel=vel)
        one = E.run(cq.generate_commands(prog1.graph(), world), placement=pl)
        err = np.linalg.norm(one.buffers["V"][:, :3] / 1e-3 - acc, axis=1) / np.linalg.norm(acc, axis=1)
        check(f"nbody {nb} x2 steps all-gather == 1 GPU; kick err {err.max():.1e}", ok and err.max() <= 1e-4)
    else:
        prog1 = W.nbody_program(nb, steps=1, pos=pos, vel=vel)
        E.run(cq.generate_commands(prog1.graph(), world), placement=pl)

    # SGEMM slice mappers (A scatter + B broadcast), both variants
    m, nn, k = 512, 384, 256
    a, b = W.sgemm_inputs(m, nn, k)
    for variant in ("ffma", "3xtf32"):
        prog = W.sgemm_program(m, nn, k, variant=variant, a=a, b=b)
        res = E.run(cq.generate_commands(prog.graph(), world), placement=pl)
        if rank == 0:
            rows = np.arange(0, m, 5)
            c, cabs = onat.sgemm_rows(a, b, rows)
            err = np.abs(res.buffers["C"][rows] - c) / cabs
            check(f"sgemm {variant} {m}x{nn}x{k} err={err.max():.2e}", err.max() <= 1e-6)

    # fused chain across ranks with peer-memory halo rows (CUDA IPC + NVLink
    # copies, device pass counters): a run, then a captured graph replayed
    # twice continuing the simulation on the device
    before = E.STATS["peer_blocks"]
    prog = W.wave_program(h, w, steps=22, kind="float32", u0=u0, up0=up0)
    sess = E.Session(cq.generate_commands(prog.graph(), world), pl)
    sess.execute(upload=True)
    sess.synchronize()
    first = sess.results()
    sess.recycle()
    sess.capture()
    sess.replay(2)
    sess.synchronize()
    again = sess.results()
    sess.close()
    if rank == 0:
        u1, up1 = onat.wave_run(u0, up0, 22, 0.25)
        u3, up3 = onat.wave_run(u0, up0, 66, 0.25)
        used = E.STATS["peer_blocks"] - before
        check(f"wave fused nodes={world} peer-memory halo rows ({used} blocks), run + 2 graph replays",
              (used > 0 or world == 1 or os.environ.get("CQ_WAVE_P2P") == "0") and dsl.same_bits(first["u"], u1) and dsl.same_bits(first["up"], up1)
              and dsl.same_bits(again["u"], u3) and dsl.same_bits(again["up"], up3))

    # magnitudes near the float32 limit in the rows a neighbour reads as halo
    # (5 rows into rank 1): the neighbour's pass must see the shared bound and
    # keep the exact form there (4u overflows where an FMA would not)
    if world > 1:
        lo1 = cq.generate_commands(W.wave_program(h, w, steps=12, kind="float32").graph(), world)
        lo1 = min(c.chunk.box.mins[0] for c in lo1.commands
                  if isinstance(c, E.ExecuteCommand) and c.node == 1)
        hu0 = np.random.default_rng(24).uniform(0, 1, (h, w)).astype(np.float32)
        hup0 = hu0.copy()
        hu0[lo1 + 5, 50:90] = np.float32(1.2e38)
        hup0[lo1 + 6, 200:220] = np.float32(-9e37)
        prog = W.wave_program(h, w, steps=12, kind="float32", c=0.3, u0=hu0, up0=hup0)
        res = E.run(cq.generate_commands(prog.graph(), world), placement=pl)
        if rank == 0:
            u, up = onat.wave_run(hu0, hup0, 12, 0.3)
            check(f"wave fused nodes={world} huge values in a neighbour's halo rows (shared bound)",
                  dsl.same_bits(res.buffers["u"], u) and dsl.same_bits(res.buffers["up"], up))

    # one node's row pushed to every other node: one in-place ncclBroadcast
    before = E.STATS["bcast"]
    res = E.run(cq.generate_commands(W.row_broadcast_program(4 * world).graph(), world), placement=pl)
    if rank == 0:
        rows, cols = 4 * world, 64
        want = ((2 * np.arange(cols, dtype=np.float32) + 1) * 3)[None, :] + np.arange(rows, dtype=np.float32)[:, None]
        check(f"row broadcast nodes={world}: one ncclBroadcast ({E.STATS['bcast'] - before}), values exact",
              E.STATS["bcast"] - before == (1 if world > 1 else 0) and np.array_equal(res.buffers["d"], want))

    dist.barrier()
    E.shutdown_distributed()
    dist.destroy_process_group()
    if rank == 0:
        print("ALL PASS" if not failures else f"FAILED: {failures}", flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
