"""Generate golden fixtures FROM THE REFERENCE (run in the build container,
where /root/reference exists):

    python tests/golden/make_golden.py

* programs.json / expected.npz -- programs (reference random workloads from
  pkg/tests/helpers.py:210-317, the bundled scenarios, a 2-D wave ping-pong and
  SAXPY) with the reference simulator's final buffers (simulator.run,
  simulator.py:101-224) and each program's reference plan signature hash at
  3 nodes;
* dot/*.dot -- reference command-graph DOT text (scheduler.py:372-392) for
  BASELINE-shaped plans;
* energy.json -- reference frequency selections and energy reports.

The GPU tests replay these on the B200 (tests/test_gpu_parity.py).
"""

import hashlib
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from progjson import program_to_json, program_from_json  # noqa: E402
from refcompat import plan_signature, ref, ref_helpers, to_mine, to_reference  # noqa: E402

import paper_2505_06022_b200 as cq  # noqa: E402
from paper_2505_06022_b200 import workloads as W  # noqa: E402


def ref_run(rbufs, rtasks, nodes):
    r = ref()
    g = r.TaskGraph(rbufs)
    for t in rtasks:
        t.id = None
        g.submit(t)
    plan = r.generate_commands(g, nodes)
    res = r.run(plan)
    return plan, res


def main():
    r = ref()
    programs = []
    arrays = {}

    def add(name, mbufs, mtasks, rbufs, rtasks, nodes=3):
        idx = len(programs)
        entry = {"name": name, "program": program_to_json(mbufs, mtasks), "nodes": nodes}
        try:
            plan, res = ref_run(rbufs, rtasks, nodes)
            plan1, res1 = ref_run(rbufs, rtasks, 1)
            entry["error"] = None
            entry["plan_sha"] = hashlib.sha256(plan_signature(plan).encode()).hexdigest()
            for bname, arr in res.buffers.items():
                assert np.array_equal(arr.view(np.uint64 if arr.dtype.kind == "f" else arr.dtype),
                                      res1.buffers[bname].view(np.uint64 if arr.dtype.kind == "f"
                                                               else arr.dtype))
                arrays[f"p{idx}__{bname}"] = arr
        except r.ClusterqError as e:
            entry["error"] = type(e).__name__
        programs.append(entry)

    # 1. reference random workloads
    for seed in (101, 103, 107, 109, 113):
        rng = random.Random(seed)
        for k in range(12):
            rbufs, rtasks = ref_helpers().random_workload(rng)
            mb, mt = to_mine(rbufs), [to_mine(t) for t in rtasks]
            add(f"random{seed}_{k}", mb, mt, rbufs, rtasks, nodes=rng.choice((2, 3, 4)))

    # 2. bundled scenarios (pkg/src/clusterq/scenarios/*.json)
    scen_dir = os.path.join(os.path.dirname(r.__file__), "scenarios")
    for fname in sorted(os.listdir(scen_dir)):
        with open(os.path.join(scen_dir, fname)) as fh:
            doc = json.load(fh)
        sc = r.scenario_from_dict(doc)
        rbufs = dict(sc.buffers) if isinstance(sc.buffers, dict) else {b.name: b for b in sc.buffers}
        rtasks = list(sc.tasks)
        mb = to_mine(rbufs)
        mt = [to_mine(t) for t in rtasks]
        add("scenario_" + fname[:-5], mb, mt, rbufs, rtasks, nodes=3)

    # 3. 2-D wave ping-pong in float64, explicit values
    for (h, w, steps, nodes) in ((40, 24, 5, 3), (33, 17, 4, 4)):
        u0 = np.random.default_rng(2).uniform(0, 1, (h, w))
        up0 = np.random.default_rng(7).uniform(0, 1, (h, w))
        prog = W.wave_program(h, w, steps=steps, kind="float64", c=0.25, u0=u0, up0=up0)
        mb = {"u": cq.Buffer("u", cq.Box.from_shape((h, w)), "float64",
                             cq.BufferInit.explicit(u0.ravel().tolist())),
              "up": cq.Buffer("up", cq.Box.from_shape((h, w)), "float64",
                              cq.BufferInit.explicit(up0.ravel().tolist()))}
        rbufs, rtasks = to_reference(mb, prog.tasks)
        add(f"wave_{h}x{w}x{steps}", mb, prog.tasks, rbufs, rtasks, nodes=nodes)

    # 4. SAXPY, reference config 1 shape scaled down (iota / constant 1)
    prog = W.saxpy_program(4096, kind="float64")
    rbufs, rtasks = to_reference(prog.buffers, prog.tasks)
    add("saxpy_4096", prog.buffers, prog.tasks, rbufs, rtasks, nodes=4)

    with open(os.path.join(HERE, "programs.json"), "w") as fh:
        json.dump(programs, fh, indent=None, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "expected.npz"), **arrays)

    # DOT fixtures of BASELINE-shaped plans
    os.makedirs(os.path.join(HERE, "dot"), exist_ok=True)
    dots = {
        "saxpy_2p24_n4": (W.saxpy_program(1 << 24, kind="float64"), 4),
        "wave_256x128_s4_n4": (W.wave_program(256, 128, steps=4, kind="float64"), 4),
        "nbody_1024_s2_n4": (W.nbody_program(1024, steps=2), 4),
        "sgemm_256_n8": (W.sgemm_program(256, 256, 256), 8),
    }
    for name, (prog, nodes) in dots.items():
        rbufs, rtasks = to_reference(prog.buffers, prog.tasks)
        g = r.TaskGraph(rbufs)
        for t in rtasks:
            g.submit(t)
        with open(os.path.join(HERE, "dot", name + ".dot"), "w") as fh:
            fh.write(r.export_command_graph(r.generate_commands(g, nodes)))

    # energy: selections and one accounting report
    dev = r.DeviceModel()
    sel = []
    for target in r.EnergyTarget:
        for t_ref in ("1/1000", "1", "7/3"):
            for beta in (0.0, 0.25, 0.5, 1.0):
                from fractions import Fraction
                f = r.select_frequency(dev, target, Fraction(t_ref), beta)
                sel.append([target.value, t_ref, beta, f])
    prog = W.saxpy_program(64, kind="float64")
    rbufs, rtasks = to_reference(prog.buffers, prog.tasks)
    plan, res = ref_run(rbufs, rtasks, 3)
    rep = r.account_energy(res.trace, plan.devices, res.makespan)
    energy = {"selections": sel,
              "trace": [[e.kind, e.node, e.command_id, str(e.start), str(e.duration), e.frequency_ghz,
                         e.task_id, e.task_name] for e in res.trace],
              "makespan": str(res.makespan),
              "per_task": [[t.task_id, str(t.energy_j), str(t.duration_s)] for t in rep.per_task],
              "per_device": [[d.node, str(d.energy_j), str(d.busy_s), str(d.idle_s)] for d in rep.per_device]}
    with open(os.path.join(HERE, "energy.json"), "w") as fh:
        json.dump(energy, fh, indent=1)
    print(f"{len(programs)} programs, {len(arrays)} arrays, {len(dots)} dot files")


if __name__ == "__main__":
    main()
