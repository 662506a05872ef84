"""JSON (de)serialisation of programs (buffers + tasks) for golden fixtures,
so programs generated from the reference in this container can be replayed on
the GPU box where the reference does not exist."""

import numpy as np

import paper_2505_06022_b200 as cq
from paper_2505_06022_b200 import kernel as K


def _ast(e):
    """AST as nested lists (exact: no text round trip, negative literals kept)."""
    if isinstance(e, K.Num):
        return ["num", e.value]
    if isinstance(e, K.Param):
        return ["param", e.name]
    if isinstance(e, K.IdComponent):
        return ["id", e.axis]
    if isinstance(e, K.Read):
        return ["read", e.accessor, list(e.offsets)]
    if isinstance(e, K.Neg):
        return ["neg", _ast(e.operand)]
    return ["bin", e.op, _ast(e.left), _ast(e.right)]


def _unast(d):
    t = d[0]
    if t == "num":
        return K.Num(d[1])
    if t == "param":
        return K.Param(d[1])
    if t == "id":
        return K.IdComponent(d[1])
    if t == "read":
        return K.Read(d[1], tuple(d[2]))
    if t == "neg":
        return K.Neg(_unast(d[1]))
    return K.BinOp(d[1], _unast(d[2]), _unast(d[3]))


def _box(b):
    return [list(b.mins), list(b.maxs)]


def _unbox(d):
    return cq.Box(d[0], d[1])


def _mapper(m):
    if isinstance(m, cq.OneToOne):
        return {"kind": "one_to_one"}
    if isinstance(m, cq.Neighborhood):
        return {"kind": "neighborhood", "radii": list(m.radii)}
    if isinstance(m, cq.All):
        return {"kind": "all"}
    if isinstance(m, cq.Slice):
        return {"kind": "slice", "axis": m.axis}
    return {"kind": "fixed", "boxes": [_box(b) for b in m.region.boxes], "dims": m.region.dims}


def _unmapper(d):
    k = d["kind"]
    if k == "one_to_one":
        return cq.OneToOne()
    if k == "neighborhood":
        return cq.Neighborhood(tuple(d["radii"]))
    if k == "all":
        return cq.All()
    if k == "slice":
        return cq.Slice(d["axis"])
    return cq.Fixed(cq.Region(d["dims"], [_unbox(b) for b in d["boxes"]]))


def program_to_json(buffers, tasks):
    bufs = []
    for name, b in buffers.items():
        init = {"kind": b.init.kind}
        if b.init.kind == "constant":
            init["value"] = b.init.value
        if b.init.kind == "values":
            init["values"] = list(b.init.values)
        bufs.append({"name": name, "extent": list(b.extent.maxs), "kind": b.element_kind, "init": init})
    ts = []
    for t in tasks:
        accs = [{"buffer": a.buffer, "mode": a.mode.value, "mapper": _mapper(a.mapper), "name": a.name}
                for a in t.accessors]
        ts.append({"name": t.name, "range": _box(t.global_range), "accessors": accs,
                   "body": {k: _ast(v) for k, v in t.body.items()},
                   "params": dict(t.params), "beta": t.beta,
                   "target": None if t.target is None else t.target.value})
    return {"buffers": bufs, "tasks": ts}


def program_from_json(d):
    buffers = {}
    for b in d["buffers"]:
        i = b["init"]
        init = cq.BufferInit(i["kind"], value=i.get("value"),
                             values=tuple(i["values"]) if "values" in i else None)
        buffers[b["name"]] = cq.Buffer(b["name"], cq.Box.from_shape(b["extent"]), b["kind"], init)
    tasks = []
    for t in d["tasks"]:
        accs = [cq.Accessor(a["buffer"], cq.AccessMode(a["mode"]), _unmapper(a["mapper"]), name=a["name"])
                for a in t["accessors"]]
        rng = _unbox(t["range"])
        body = {k: _unast(v) for k, v in t["body"].items()}
        tgt = None if t["target"] is None else cq.EnergyTarget(t["target"])
        tasks.append(cq.Task(t["name"], rng, accs, body, params=dict(t["params"]), beta=t["beta"],
                             target=tgt))
    return buffers, tasks


def graph_of(buffers, tasks):
    g = cq.TaskGraph(buffers)
    for t in tasks:
        g.submit(t)
    return g


def save_arrays(path, arrays):
    np.savez_compressed(path, **arrays)


def load_arrays(path):
    with np.load(path) as z:
        return {k: z[k] for k in z.files}
