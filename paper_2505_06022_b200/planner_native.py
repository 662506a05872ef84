"""Native planner binding: ``generate_commands`` on the C++ core
(csrc/cq_plan.cpp) returning the *same* ``Plan`` objects as the Python
planner (scheduler.py).  Host-only code -- it needs libcq.so but no GPU.

The graph (validation, conflict edges) stays in Python (``TaskGraph.submit``
is the user-facing queue); the wire format carries buffers, task ranges,
accessors/mappers and each task's predecessor list.  Frequencies are attached
here with the reference's exact-rational selection (energy.py:93-106),
memoised per (device, target, chunk volume, beta).
"""

import ctypes
from fractions import Fraction

import numpy as np

from . import _native as N
from .energy import resolve_target
from .synergy import select_for_task
from .model import AccessMode, All, Fixed, Neighborhood, OneToOne, Slice
from .region import Region, _raw as _mk, _blank as _new, _put as _set
from .scheduler import (AwaitPushCommand, Chunk, ExecuteCommand, Plan, PushCommand,
                        _resolve_devices)
from .errors import NativeError, ValidationError


def _encode(graph):
    names = list(graph.buffers)
    index = {n: i for i, n in enumerate(names)}
    w = [len(names)]
    for n in names:
        b = graph.buffers[n]
        w += [b.dims, *b.extent.maxs, 1 if b.init.is_initialized else 0, b.itemsize]
    tasks = graph.tasks
    tindex = {t.id: i for i, t in enumerate(tasks)}
    w.append(len(tasks))
    for t in tasks:
        preds = [tindex[p] for p in graph.predecessors(t.id)]
        w += [t.dims, *t.global_range.maxs, len(preds), *preds, len(t.accessors)]
        for a in t.accessors:
            w += [index[a.buffer], 0 if a.mode is AccessMode.READ else 1]
            m = a.mapper
            if isinstance(m, OneToOne):
                w.append(0)
            elif isinstance(m, Neighborhood):
                w += [1, *m.radii]
            elif isinstance(m, All):
                w.append(2)
            elif isinstance(m, Slice):
                w += [3, m.axis]
            elif isinstance(m, Fixed):
                w += [4, len(m.region.boxes)]
                for bx in m.region.boxes:
                    w += [*bx.mins, *bx.maxs]
            else:
                raise ValidationError(f"native planner: unknown mapper {m!r}")
    return names, np.asarray(w, dtype=np.int64)


class _Reader:
    __slots__ = ("a", "i")

    def __init__(self, a):
        self.a = a
        self.i = 0

    def next(self):
        v = self.a[self.i]
        self.i += 1
        return v

    def take(self, n):
        v = self.a[self.i:self.i + n]
        self.i += n
        return v

    def region(self, d):
        nb = self.next()
        boxes = []
        for _ in range(nb):
            lo = tuple(self.take(d))
            hi = tuple(self.take(d))
            boxes.append(_mk(lo, hi))
        r = _new(Region)
        _set(r, "dims", d)
        _set(r, "boxes", tuple(boxes))
        return r


def generate_commands_native(graph, node_count, devices=None, queue_target=None):
    from .energy import EnergyTarget
    if queue_target is None:
        queue_target = EnergyTarget.MAX_PERF
    if node_count < 1:
        raise ValidationError("node count must be at least 1")
    devices = _resolve_devices(devices, node_count)
    names, words = _encode(graph)
    lib = N.load_host()
    out = ctypes.POINTER(ctypes.c_int64)()
    n_out = ctypes.c_int64()
    status = lib.cq_plan_generate(words.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), words.size,
                                  node_count, ctypes.byref(out), ctypes.byref(n_out))
    if status != N.CQ_OK:
        raise NativeError("cq_plan_generate: " + lib.cq_last_error().decode(errors="replace"), status)
    try:
        flat = np.ctypeslib.as_array(out, shape=(n_out.value,)).tolist()
    finally:
        lib.cq_plan_free(out)

    rd = _Reader(flat)
    tasks = graph.tasks
    dims_of = [graph.buffers[n].dims for n in names]
    ebytes = [graph.buffers[n].itemsize for n in names]
    freq_memo = {}
    commands = []
    for cid in range(rd.next()):
        kind = rd.next()
        deps = tuple(rd.take(rd.next()))
        if kind == 0:
            ti = rd.next()
            node = rd.next()
            task = tasks[ti]
            d = task.dims
            lo = tuple(rd.take(d))
            hi = tuple(rd.take(d))
            box = _mk(lo, hi)
            reads = []
            for _ in range(rd.next()):
                acc = task.accessors[rd.next()]
                reads.append((acc.name, acc.buffer, rd.region(graph.buffers[acc.buffer].dims)))
            writes = []
            for _ in range(rd.next()):
                acc = task.accessors[rd.next()]
                reg = rd.region(graph.buffers[acc.buffer].dims)
                writes.append((acc.name, acc.buffer, reg, rd.next()))
            dev = devices[node]
            target = resolve_target(queue_target, task.target)
            vol = box.volume()
            key = (id(dev), target, vol, task.beta, task.name)
            f = freq_memo.get(key)
            if f is None:
                f = freq_memo[key] = select_for_task(dev, target, Fraction(vol) / Fraction(dev.throughput_ref), task)
            commands.append(ExecuteCommand(id=cid, deps=deps, chunk=Chunk(task.id, box, node),
                                           frequency_ghz=f, reads=tuple(reads), writes=tuple(writes)))
        elif kind == 1:
            src, dst, b, version = rd.next(), rd.next(), rd.next(), rd.next()
            commands.append(PushCommand(id=cid, deps=deps, src=src, dst=dst, buffer=names[b],
                                        region=rd.region(dims_of[b]), version=version,
                                        element_bytes=ebytes[b]))
        else:
            dst, b, version, push_id = rd.next(), rd.next(), rd.next(), rd.next()
            commands.append(AwaitPushCommand(id=cid, deps=deps, dst=dst, buffer=names[b],
                                             region=rd.region(dims_of[b]), version=version,
                                             push_id=push_id))
    final = {}
    for bi, name in enumerate(names):
        entries = []
        for _ in range(rd.next()):
            version = rd.next()
            holders = frozenset(rd.take(rd.next()))
            entries.append((rd.region(dims_of[bi]), version, holders))
        final[name] = entries
    return Plan(graph=graph, node_count=node_count, commands=commands, devices=devices,
                queue_target=queue_target, final_locations=final)
