"""Test-side bridge to the read-only reference (clusterq) in this container.

Used ONLY by tests and by tests/golden/make_golden.py to pin the oracle and the
planner against the real reference.  Nothing here runs on the GPU box (the
reference does not exist there; tests needing it carry @pytest.mark.reference).
"""

import importlib.util
import os
import sys

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"

_cache = {}


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "clusterq"))


def ref():
    """The reference ``clusterq`` package (imported read-only)."""
    if "clusterq" not in _cache:
        os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
        sys.dont_write_bytecode = True
        if REF_SRC not in sys.path:
            sys.path.append(REF_SRC)
        import clusterq  # noqa: E402
        _cache["clusterq"] = clusterq
    return _cache["clusterq"]


def ref_helpers():
    """The reference's tests/helpers.py (random_workload, check_plan)."""
    if "helpers" not in _cache:
        ref()
        spec = importlib.util.spec_from_file_location("ref_helpers", os.path.join(REF_TESTS, "helpers.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _cache["helpers"] = mod
    return _cache["helpers"]


# ------------------------------------------------------------ conversions

def to_mine(obj):
    """Convert reference model objects to this package's equivalents."""
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import kernel as K
    r = ref()
    rk = sys.modules["clusterq.kernel"]
    rm = sys.modules["clusterq.model"]
    if isinstance(obj, r.Box):
        return cq.Box(obj.mins, obj.maxs)
    if isinstance(obj, r.Region):
        return cq.Region(obj.dims, [to_mine(b) for b in obj.boxes])
    if isinstance(obj, rk.Num):
        return K.Num(obj.value)
    if isinstance(obj, rk.Param):
        return K.Param(obj.name)
    if isinstance(obj, rk.IdComponent):
        return K.IdComponent(obj.axis)
    if isinstance(obj, rk.Read):
        return K.Read(obj.accessor, tuple(obj.offsets))
    if isinstance(obj, rk.Neg):
        return K.Neg(to_mine(obj.operand))
    if isinstance(obj, rk.BinOp):
        return K.BinOp(obj.op, to_mine(obj.left), to_mine(obj.right))
    if isinstance(obj, rm.OneToOne):
        return cq.OneToOne()
    if isinstance(obj, rm.Neighborhood):
        return cq.Neighborhood(obj.radii)
    if isinstance(obj, rm.All):
        return cq.All()
    if isinstance(obj, rm.Slice):
        return cq.Slice(obj.axis)
    if isinstance(obj, rm.Fixed):
        return cq.Fixed(to_mine(obj.region))
    if isinstance(obj, rm.BufferInit):
        return cq.BufferInit(obj.kind, value=obj.value, values=obj.values)
    if isinstance(obj, rm.Buffer):
        return cq.Buffer(obj.name, to_mine(obj.extent), obj.element_kind, to_mine(obj.init))
    if isinstance(obj, rm.Accessor):
        mode = cq.AccessMode.READ if obj.mode is rm.AccessMode.READ else cq.AccessMode.WRITE
        return cq.Accessor(obj.buffer, mode, to_mine(obj.mapper), name=obj.name)
    if isinstance(obj, rm.Task):
        tgt = None if obj.target is None else cq.EnergyTarget(obj.target.value)
        return cq.Task(name=obj.name, global_range=to_mine(obj.global_range),
                       accessors=[to_mine(a) for a in obj.accessors],
                       body={k: to_mine(v) for k, v in obj.body.items()},
                       params=dict(obj.params), beta=obj.beta, target=tgt)
    if isinstance(obj, r.DeviceModel):
        return cq.DeviceModel(obj.levels_ghz, obj.f_ref_ghz, obj.p_static_w, obj.p_dyn_ref_w,
                              obj.alpha_exp, obj.throughput_ref, obj.node)
    if isinstance(obj, dict):
        return {k: to_mine(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return type(obj)(to_mine(v) for v in obj)
    raise TypeError(f"cannot convert {type(obj)!r}")


def plan_signature(plan, with_bytes=True):
    """Backend-neutral text form of a plan: every command field plus final
    locations.  Two planners agree iff their signatures are equal."""
    out = []
    for c in plan.commands:
        kind = type(c).__name__
        deps = ",".join(str(d) for d in c.deps)
        if kind == "ExecuteCommand":
            reads = ";".join(f"{a}:{b}:{r}" for a, b, r in c.reads)
            writes = ";".join(f"{a}:{b}:{r}:v{v}" for a, b, r, v in c.writes)
            out.append(f"{c.id} X t{c.chunk.task_id} {c.chunk.box} n{c.chunk.node} "
                       f"f{c.frequency_ghz!r} d[{deps}] R[{reads}] W[{writes}]")
        elif kind == "PushCommand":
            out.append(f"{c.id} P {c.buffer} {c.region} v{c.version} n{c.src}->n{c.dst} "
                       f"d[{deps}]" + (f" b{c.bytes}" if with_bytes else ""))
        else:
            out.append(f"{c.id} A {c.buffer} {c.region} v{c.version} n{c.dst} "
                       f"p{c.push_id} d[{deps}]")
    for name in sorted(plan.final_locations):
        for region, version, holders in plan.final_locations[name]:
            out.append(f"F {name} {region} v{version} h{sorted(holders)}")
    return "\n".join(out) + "\n"


def to_reference(buffers, tasks):
    """Convert this package's program to reference objects for planning.

    float32 becomes float64 (the reference has no 4-byte kind; only push byte
    counts differ), array inits become zeros (planning needs only
    ``is_initialized``), native bodies become a placeholder expression that
    reads a one_to_one accessor (the reference DSL cannot express them,
    SPEC.md:181) -- accessors and mappers, i.e. the data requirements, are
    unchanged."""
    import paper_2505_06022_b200 as cq
    from paper_2505_06022_b200 import kernel as K
    r = ref()
    rk = sys.modules["clusterq.kernel"]

    def box(b):
        return r.Box(b.mins, b.maxs)

    def region(g):
        return r.Region(g.dims, [box(b) for b in g.boxes])

    def mapper(m):
        if isinstance(m, cq.OneToOne):
            return r.OneToOne()
        if isinstance(m, cq.Neighborhood):
            return r.Neighborhood(m.radii)
        if isinstance(m, cq.All):
            return r.All()
        if isinstance(m, cq.Slice):
            return r.Slice(m.axis)
        return r.Fixed(region(m.region))

    def expr(e):
        if isinstance(e, K.Num):
            return rk.Num(e.value)
        if isinstance(e, K.Param):
            return rk.Param(e.name)
        if isinstance(e, K.IdComponent):
            return rk.IdComponent(e.axis)
        if isinstance(e, K.Read):
            return rk.Read(e.accessor, e.offsets)
        if isinstance(e, K.Neg):
            return rk.Neg(expr(e.operand))
        return rk.BinOp(e.op, expr(e.left), expr(e.right))

    rbufs = {}
    for name, b in buffers.items():
        init = b.init
        if init.kind == "array":
            rinit = r.BufferInit.zeros()
        else:
            rinit = r.BufferInit(init.kind, value=init.value, values=init.values)
        kind = "float64" if b.element_kind == "float32" else b.element_kind
        rbufs[name] = r.Buffer(name, box(b.extent), kind, rinit)
    rtasks = []
    for t in tasks:
        accs = []
        for a in t.accessors:
            mode = r.AccessMode.READ if a.mode is cq.AccessMode.READ else r.AccessMode.WRITE
            accs.append(r.Accessor(a.buffer, mode, mapper(a.mapper), name=a.name))
        if isinstance(t.body, cq.NativeKernel):
            o2o = next(a for a in t.accessors
                       if a.mode is cq.AccessMode.READ and isinstance(a.mapper, cq.OneToOne)) \
                if any(a.mode is cq.AccessMode.READ and isinstance(a.mapper, cq.OneToOne)
                       for a in t.accessors) else None
            leaf = rk.Read(o2o.name, (0,) * t.dims) if o2o is not None else rk.Num(0.0)
            body = {a.name: leaf for a in t.accessors if a.mode is cq.AccessMode.WRITE}
        else:
            body = {k: expr(v) for k, v in t.body.items()}
        tgt = None if t.target is None else r.EnergyTarget(t.target.value)
        rtasks.append(r.Task(name=t.name, global_range=box(t.global_range), accessors=accs,
                             body=body, params=dict(t.params), beta=t.beta, target=tgt))
    return rbufs, rtasks


def to_reference_plan(plan, rgraph):
    """This package's ``Plan`` as the reference's command objects over the
    reference graph ``rgraph`` (built from the same program, so task ids
    agree), for the reference's own ``check_plan`` (tests/helpers.py:59-165)."""
    r = ref()
    rs = sys.modules["clusterq.scheduler"]

    def box(b):
        return r.Box(b.mins, b.maxs)

    def region(g):
        return r.Region(g.dims, [box(b) for b in g.boxes])

    cmds = []
    for c in plan.commands:
        kind = type(c).__name__
        if kind == "ExecuteCommand":
            cmds.append(rs.ExecuteCommand(c.id, tuple(c.deps), rs.Chunk(c.chunk.task_id, box(c.chunk.box),
                                                                          c.chunk.node),
                                          c.frequency_ghz, tuple((a, b, region(g)) for a, b, g in c.reads),
                                          tuple((a, b, region(g), v) for a, b, g, v in c.writes)))
        elif kind == "PushCommand":
            cmds.append(rs.PushCommand(c.id, tuple(c.deps), c.src, c.dst, c.buffer, region(c.region), c.version))
        else:
            cmds.append(rs.AwaitPushCommand(c.id, tuple(c.deps), c.dst, c.buffer, region(c.region), c.version,
                                            c.push_id))
    finals = {name: [(region(g), v, set(h)) for g, v, h in entries]
              for name, entries in plan.final_locations.items()}
    return rs.Plan(rgraph, plan.node_count, cmds, [], r.EnergyTarget.MAX_PERF, finals)


def drop_push(plan, push):
    """``plan`` without ``push`` and its AwaitPush (and the deps on them) --
    the negative control: a plan that loses one transfer."""
    import dataclasses
    gone = {push.id} | {c.id for c in plan.commands
                        if type(c).__name__ == "AwaitPushCommand" and c.push_id == push.id}
    cmds = []
    for c in plan.commands:
        if c.id in gone:
            continue
        cmds.append(dataclasses.replace(c, deps=tuple(d for d in c.deps if d not in gone)))
    return dataclasses.replace(plan, commands=cmds)
