"""The BASELINE programs, written against the drop-in API.

Each builder returns a ``Program`` (buffers + tasks) exactly as a user of the
reference API would write it; ``Program.graph()`` submits the tasks to a fresh
``TaskGraph``.  Shapes and synthetic inputs follow SURVEY.md §8(d):

* SAXPY: ``z[i] = alpha * x[i] + y[i]`` -- the reference's bundled
  scenario body (pkg/src/clusterq/scenarios/saxpy.json:15).
* 2-D wave: Celerity-style leapfrog ping-pong, ``u`` read through
  ``neighborhood(1,1)``, previous field read one_to_one, written in place;
  body (evaluated with kernel.py:291-331 operator order)
  ``2*u - upr + c*(u[N] + u[S] + u[W] + u[E] - 4*u)`` with edge clamping
  (model.py:442-446).
* N-body: ``kick`` (all-pairs acceleration, ``all`` mapper on positions ->
  all-gather) then ``drift`` (one_to_one), two tasks per step.
* matmul: ``C = A . B`` with ``slice(1)`` on A and ``slice(0)`` on B.
"""

import dataclasses
from dataclasses import dataclass

import numpy as np

from .graph import TaskGraph
from .kernel import parse_kernel
from .model import (Accessor, AccessMode, All, Buffer, BufferInit, NativeKernel,
                    Neighborhood, OneToOne, Slice, Task)
from .region import Box

R, W = AccessMode.READ, AccessMode.WRITE

SAXPY_BODY = "alpha * x[i] + y[i]"
WAVE_BODY = ("2 * u[i.0, i.1] - upr[i.0, i.1] + c * (u[i.0-1, i.1] + u[i.0+1, i.1] "
             "+ u[i.0, i.1-1] + u[i.0, i.1+1] - 4 * u[i.0, i.1])")


@dataclass
class Program:
    name: str
    buffers: dict
    tasks: list

    def graph(self) -> TaskGraph:
        g = TaskGraph(self.buffers)
        for t in self.tasks:
            g.submit(dataclasses.replace(t, id=None))
        return g


# ---------------------------------------------------------------- SAXPY

def saxpy_inputs(n, kind="float32", seed=None):
    """Reference inputs (x = iota, y = 1) or U[-1,1) with seeds 0 / 1."""
    dt = np.float32 if kind == "float32" else np.float64
    if seed is None:
        return None, None
    x = np.random.default_rng(seed).uniform(-1, 1, n).astype(dt)
    y = np.random.default_rng(seed + 1).uniform(-1, 1, n).astype(dt)
    return x, y


def saxpy_program(n, alpha=2.0, kind="float32", x=None, y=None, chunks=None) -> Program:
    ext = Box.from_shape((n,))
    bufs = {
        "x": Buffer("x", ext, kind, BufferInit.iota() if x is None else BufferInit.array(x)),
        "y": Buffer("y", ext, kind, BufferInit.constant(1) if y is None else BufferInit.array(y)),
        "z": Buffer("z", ext, kind, BufferInit.zeros()),
    }
    body = {"z": parse_kernel(SAXPY_BODY, {"x": 1, "y": 1}, {"alpha"}, 1)}
    task = Task("saxpy", ext, [Accessor("x", R), Accessor("y", R), Accessor("z", W)], body,
                params={"alpha": alpha})
    return Program("saxpy", bufs, [task])


# ------------------------------------------------------------------ wave

def wave_pulse(h, w, kind="float32"):
    """Gaussian pulse exp(-((i-H/2)^2 + (j-W/2)^2) / (2 (W/16)^2))."""
    dt = np.float32 if kind == "float32" else np.float64
    i = np.arange(h, dtype=np.float64)[:, None] - h / 2
    j = np.arange(w, dtype=np.float64)[None, :] - w / 2
    s = (w / 16.0) ** 2
    return np.exp(-(i * i + j * j) / (2 * s)).astype(dt)


def wave_task(step, h, w, c):
    """Task for time step ``step``: even steps advance buffer ``up`` from
    ``u``, odd steps advance ``u`` from ``up`` (ping-pong)."""
    cur, prev = ("u", "up") if step % 2 == 0 else ("up", "u")
    ext = Box.from_shape((h, w))
    body = {"out": parse_kernel(WAVE_BODY, {"u": 2, "upr": 2}, {"c"}, 2)}
    return Task(f"wave{step}", ext,
                [Accessor(cur, R, Neighborhood((1, 1)), name="u"),
                 Accessor(prev, R, OneToOne(), name="upr"),
                 Accessor(prev, W, name="out")],
                body, params={"c": c})


def wave_program(h, w, steps=100, kind="float32", c=0.25, u0=None, up0=None) -> Program:
    ext = Box.from_shape((h, w))
    if u0 is None:
        u0 = wave_pulse(h, w, kind)
    if up0 is None:
        up0 = u0
    bufs = {"u": Buffer("u", ext, kind, BufferInit.array(u0)),
            "up": Buffer("up", ext, kind, BufferInit.array(up0))}
    return Program("wave", bufs, [wave_task(s, h, w, c) for s in range(steps)])


def wave_result_buffer(steps) -> str:
    """Buffer holding the newest field after ``steps`` steps."""
    return "up" if steps % 2 == 1 else "u"


# ---------------------------------------------------------------- N-body

def nbody_inputs(n, seed=3):
    """Positions uniform in the unit ball (seed 3), masses U[0.5,1.5) (seed 4),
    zero velocities; rows (x, y, z, m) and (vx, vy, vz, 0)."""
    g = np.random.default_rng(seed)
    v = g.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    r = g.uniform(0, 1, n) ** (1.0 / 3.0)
    pos = np.empty((n, 4), np.float32)
    pos[:, :3] = v * r[:, None]
    pos[:, 3] = np.random.default_rng(seed + 1).uniform(0.5, 1.5, n)
    vel = np.zeros((n, 4), np.float32)
    return pos, vel


def nbody_program(n, steps=1, eps2=1e-2, dt=1e-3, pos=None, vel=None) -> Program:
    if pos is None or vel is None:
        pos, vel = nbody_inputs(n)
    ext = Box.from_shape((n, 4))
    bufs = {"P": Buffer("P", ext, "float32", BufferInit.array(pos)),
            "V": Buffer("V", ext, "float32", BufferInit.array(vel))}
    tasks = []
    for s in range(steps):
        tasks.append(Task(f"kick{s}", ext,
                          [Accessor("P", R, All(), name="pos"),
                           Accessor("V", R, OneToOne(), name="vel_in"),
                           Accessor("V", W, name="vel")],
                          NativeKernel("nbody.kick"), params={"eps2": eps2, "dt": dt}))
        tasks.append(Task(f"drift{s}", ext,
                          [Accessor("P", R, OneToOne(), name="pos_in"),
                           Accessor("V", R, OneToOne(), name="vel"),
                           Accessor("P", W, name="pos")],
                          NativeKernel("nbody.drift"), params={"dt": dt}))
    return Program("nbody", bufs, tasks)


# ---------------------------------------------------------------- matmul

def sgemm_inputs(m, n, k, seed=5):
    a = np.random.default_rng(seed).uniform(-1, 1, (m, k)).astype(np.float32)
    b = np.random.default_rng(seed + 1).uniform(-1, 1, (k, n)).astype(np.float32)
    return a, b


def sgemm_program(m, n, k, variant="3xtf32", a=None, b=None) -> Program:
    if a is None or b is None:
        a, b = sgemm_inputs(m, n, k)
    bufs = {"A": Buffer("A", Box.from_shape((m, k)), "float32", BufferInit.array(a)),
            "B": Buffer("B", Box.from_shape((k, n)), "float32", BufferInit.array(b)),
            "C": Buffer("C", Box.from_shape((m, n)), "float32", BufferInit.uninitialized())}
    task = Task("sgemm", Box.from_shape((m, n)),
                [Accessor("A", R, Slice(1), name="a"), Accessor("B", R, Slice(0), name="b"),
                 Accessor("C", W, name="c")],
                NativeKernel("sgemm", variant))
    return Program("sgemm", bufs, [task])


# --------------------------------------------------------- row broadcast

def row_broadcast_program(rows, cols=64, kind="float32") -> Program:
    """One row ``c`` written by node 0 alone (a one-row task), then read in
    full by every node's chunk of a ``rows``-row task through an 'all'
    mapper: node 0 pushes the row to every other node (one ncclBroadcast
    across ranks).  d[i, j] = (2 a_j + 1) * 3 + i with a = iota."""
    one, grid = Box.from_shape((1, cols)), Box.from_shape((rows, cols))
    bufs = {"a": Buffer("a", one, kind, BufferInit.iota()),
            "c": Buffer("c", one, kind, BufferInit.zeros()),
            "d": Buffer("d", grid, kind, BufferInit.zeros())}
    make = Task("make", one, [Accessor("a", R), Accessor("c", W)],
                {"c": parse_kernel("a[i.0, i.1] * 2 + 1", {"a": 2}, set(), 2)})
    use = Task("use", grid, [Accessor("c", R, All()), Accessor("d", W)],
               {"d": parse_kernel("c[i.0, i.1] * 3 + i.0", {"c": 2}, set(), 2)})
    return Program("row_broadcast", bufs, [make, use])

