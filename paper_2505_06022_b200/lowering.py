"""Kernel selection for Execute commands: which sm_100a kernel runs a task
body, with which operands, and whether it may run in place.

The reference evaluates every body per cell in Python
(pkg/src/clusterq/simulator.py:151-158 -> kernel.py:291-331).  Here a body is
bound once per task to one of:

* ``saxpy``  -- ``a * x[i] + y[i]`` (scenarios/saxpy.json:15) on contiguous
  cells: ``cq_saxpy``;
* ``wave5``  -- the 2-D 5-point leapfrog body: ``cq_wave5``;
* ``native`` -- a ``NativeKernel`` (N-body, sgemm);
* ``expr``   -- anything else: the postfix program runs on the device
  interpreter ``cq_expr_eval`` with the reference's clamp + mapper check.

All four produce the reference's per-operator rounding (the specialised
kernels implement exactly the recognised tree), so the choice never changes
results -- tests/test_gpu_parity.py cross-checks fast paths against the
interpreter.
"""

import os
from dataclasses import dataclass, field

from . import kernel as K
from .model import AccessMode, NativeKernel, collect_read_offsets

# Specialised kernels for recognised bodies; tests switch this off to check
# that the interpreter and the fast paths agree bit for bit.
FAST_PATHS = os.environ.get("CQ_FAST_PATHS", "1") == "1"


@dataclass
class Binding:
    kind: str                      # saxpy | wave5 | native | expr
    args: dict = field(default_factory=dict)
    programs: tuple = ()           # (write accessor name, Program) for expr
    snapshot: frozenset = frozenset()  # read accessor names needing a snapshot


def _is_scalar(e):
    return isinstance(e, (K.Num, K.Param))


def _scalar_value(e, params):
    return float(e.value if isinstance(e, K.Num) else params[e.name])


def _read(e, offsets=None):
    if not isinstance(e, K.Read):
        return None
    if offsets is not None and tuple(e.offsets) != tuple(offsets):
        return None
    return e.accessor


def match_saxpy(expr, params):
    """``s * X[0] + Y[0]`` -> (alpha, x accessor, y accessor) or None."""
    if not (isinstance(expr, K.BinOp) and expr.op == "+"):
        return None
    mul = expr.left
    if not (isinstance(mul, K.BinOp) and mul.op == "*" and _is_scalar(mul.left)):
        return None
    x = _read(mul.right)
    y = _read(expr.right)
    if x is None or y is None or any(mul.right.offsets) or any(expr.right.offsets):
        return None
    return mul.left, x, y


def match_wave5(expr, params):
    """``((k2*u) - p) + (c*((((u[-1,0] + u[1,0]) + u[0,-1]) + u[0,1]) - (k4*u)))``
    -> dict(u, upr, c, k2, k4) or None.  Operator order is part of the match:
    only this exact tree is routed to ``cq_wave5``."""
    def binop(e, op):
        return isinstance(e, K.BinOp) and e.op == op
    if not binop(expr, "+") or not binop(expr.left, "-") or not binop(expr.right, "*"):
        return None
    k2u = expr.left.left
    if not binop(k2u, "*") or not _is_scalar(k2u.left):
        return None
    u = _read(k2u.right, (0, 0))
    upr = _read(expr.left.right, (0, 0))
    c = expr.right.left
    lap = expr.right.right
    if u is None or upr is None or not _is_scalar(c) or not binop(lap, "-"):
        return None
    k4u = lap.right
    if not binop(k4u, "*") or not _is_scalar(k4u.left) or _read(k4u.right, (0, 0)) != u:
        return None
    s3 = lap.left
    if not (binop(s3, "+") and binop(s3.left, "+") and binop(s3.left.left, "+")):
        return None
    taps = [s3.left.left.left, s3.left.left.right, s3.left.right, s3.right]
    want = [(-1, 0), (1, 0), (0, -1), (0, 1)]
    if any(_read(t, o) != u for t, o in zip(taps, want)):
        return None
    return {"u": u, "upr": upr, "c": _scalar_value(c, params),
            "k2": _scalar_value(k2u.left, params), "k4": _scalar_value(k4u.left, params)}


def bind_task(task, buffers) -> Binding:
    """Choose the kernel for ``task`` (cached by the executor per task id)."""
    if isinstance(task.body, NativeKernel):
        return Binding("native", {"name": task.body.name, "variant": task.body.variant})

    accs = {a.name: a for a in task.accessors}
    written = {a.buffer for a in task.writes()}
    offsets = collect_read_offsets(task)
    # A read of a buffer this task writes is safe in place only at offset 0
    # (the same thread reads the cell before writing it); otherwise the
    # executor snapshots the read region first (reference: reads observe
    # pre-task state, simulator.py:138-145).
    snap = frozenset(name for name, offs in offsets.items()
                     if accs[name].buffer in written and any(any(o) for o in offs))

    writes = task.writes()
    if FAST_PATHS and len(writes) == 1 and not snap:
        w = writes[0]
        kind = buffers[w.buffer].element_kind
        expr = task.body[w.name]
        sx = match_saxpy(expr, task.params)
        if sx is not None:
            a, x, y = sx
            if all(buffers[accs[n].buffer].element_kind == kind for n in (x, y)):
                av = a.value if isinstance(a, K.Num) else task.params[a.name]
                return Binding("saxpy", {"alpha": av, "x": x, "y": y, "out": w.name})
        if task.dims == 2 and kind in ("float32", "float64"):
            wv = match_wave5(expr, task.params)
            if wv is not None and buffers[accs[wv["u"]].buffer].dims == 2 \
                    and buffers[accs[wv["upr"]].buffer].dims == 2:
                wv["out"] = w.name
                return Binding("wave5", wv)

    programs = []
    for w in writes:
        kind = buffers[w.buffer].element_kind
        programs.append((w.name, K.lower(task.body[w.name], task.params, kind)))
    return Binding("expr", {}, tuple(programs), snap)


def read_accessors(task):
    return [a for a in task.accessors if a.mode is AccessMode.READ]
