"""Multi-rank parity on the GPUs of one box: one process per GPU via torchrun,
NCCL send/recv groups between ranks (skipped on a 1-GPU box)."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_torchrun_ranks_match_oracle():
    n = min(_gpus(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "scripts", "mgpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "ALL PASS" in r.stdout


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_one_process_several_gpus_matches_oracle():
    """Nodes spread over the GPUs of one process (peer box copies, cross-
    device events): fused and per-step wave, SAXPY and N-body."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import executor as E, workloads as W
    from oracle import dsl
    from oracle import native as onat
    devs = tuple(range(min(_gpus(), 4)))
    pl = E.Placement(1, 0, devs)
    h, w = 515, 384
    u0 = np.random.default_rng(2).uniform(0, 1, (h, w)).astype(np.float32)
    up0 = np.random.default_rng(3).uniform(0, 1, (h, w)).astype(np.float32)
    for steps, fuse in ((22, "1"), (9, "0")):
        os.environ["CQ_WAVE_FUSE"] = fuse
        try:
            for nodes in (len(devs), 2 * len(devs) + 1):
                prog = W.wave_program(h, w, steps=steps, kind="float32", u0=u0, up0=up0)
                res = E.run(cq.generate_commands(prog.graph(), nodes), placement=pl)
                u, up = onat.wave_run(u0, up0, steps, 0.25)
                assert dsl.same_bits(res.buffers["u"], u) and dsl.same_bits(res.buffers["up"], up), (steps, nodes)
        finally:
            os.environ.pop("CQ_WAVE_FUSE")
    n = (1 << 20) + 3
    x, y = W.saxpy_inputs(n, "float32", seed=0)
    res = E.run(cq.generate_commands(W.saxpy_program(n, kind="float32", x=x, y=y).graph(), 4), placement=pl)
    assert dsl.same_bits(res.buffers["z"], onat.saxpy(2.0, x, y))
    pos, vel = W.nbody_inputs(2048)
    outs = [E.run(cq.generate_commands(W.nbody_program(2048, steps=2, pos=pos, vel=vel).graph(), k),
                  placement=pl).buffers for k in (1, 3)]
    assert dsl.same_bits(outs[0]["P"], outs[1]["P"]) and dsl.same_bits(outs[0]["V"], outs[1]["V"])
