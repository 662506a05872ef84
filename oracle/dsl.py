"""TEST INFRASTRUCTURE ONLY -- serial restatement of the reference's program
semantics (the oracle for final buffer contents).

The reference defines distributed correctness as "final buffers at any node
count equal the 1-node run bit-exactly" (SPEC.md:343,
pkg/src/clusterq/scenario.py:611-628).  The 1-node run executes each task over
its whole range, every read seeing pre-task state (simulator.py:138-145),
each cell evaluated by eval_kernel (kernel.py:291-331) through ReadView
(model.py:442-453).  This module restates that with numpy, vectorised per AST
node (one numpy operator per DSL operator keeps one rounding per operator):

* float64: numpy float64 elementwise ops == Python float ops (IEEE);
* float32: numpy float32 elementwise ops (one binary32 rounding per op);
* int64: wrapping arithmetic; truncating division; division by zero raises
  EvalError (kernel.py:315-321);
* reads: index + offset per buffer axis (buffer axis j <- kernel axis j),
  clamped to the extent, then checked against the accessor's mapped region
  (MapperViolationError).

It consumes the program objects of the product API (buffers, tasks, AST
nodes) but implements every semantic rule itself.
"""

import numpy as np

_DT = {"float64": np.float64, "float32": np.float32, "int64": np.int64}


class OracleError(Exception):
    def __init__(self, kind, message):
        super().__init__(message)
        self.kind = kind  # "eval" | "mapper"


def initial_array(buf):
    """Initial contents (BufferInit.materialize, model.py:63-74)."""
    dt = _DT[buf.element_kind]
    shape = tuple(buf.extent.maxs)
    init = buf.init
    n = int(np.prod(shape))
    if init.kind == "iota":
        return np.arange(n, dtype=np.int64).astype(dt).reshape(shape)
    if init.kind == "constant":
        return np.full(shape, init.value, dtype=dt)
    if init.kind == "values":
        return np.array(init.values, dtype=dt).reshape(shape)
    if init.kind == "array":
        return np.array(init.data, dtype=dt).reshape(shape)
    return np.zeros(shape, dtype=dt)


def _mapped_mask(mapper, rng_lo, rng_hi, extent_shape):
    """Boolean mask of the mapper image of the full kernel range
    (model.py:135-231), clamped to the extent."""
    name = type(mapper).__name__
    d = len(extent_shape)
    mask = np.zeros(extent_shape, dtype=bool)
    if name == "All":
        mask[...] = True
        return mask
    if name == "Fixed":
        for box in mapper.region.boxes:
            sl = tuple(slice(max(a, 0), min(b, e)) for a, b, e in zip(box.mins, box.maxs, extent_shape))
            if all(s.start < s.stop for s in sl):
                mask[sl] = True
        return mask
    lo = list(rng_lo[:d])
    hi = list(rng_hi[:d])
    if name == "Neighborhood":
        lo = [a - r for a, r in zip(lo, mapper.radii)]
        hi = [b + r for b, r in zip(hi, mapper.radii)]
    elif name == "Slice":
        lo[mapper.axis] = 0
        hi[mapper.axis] = extent_shape[mapper.axis]
    sl = tuple(slice(max(a, 0), min(b, e)) for a, b, e in zip(lo, hi, extent_shape))
    if all(s.start < s.stop for s in sl):
        mask[sl] = True
    return mask


def _wrap_div(a, b):
    """int64 truncating division with the reference's sign rule."""
    if np.any(b == 0):
        raise OracleError("eval", "integer division by zero")
    ua = np.where(a < 0, (-(a.astype(np.uint64))), a.astype(np.uint64))
    ub = np.where(b < 0, (-(b.astype(np.uint64))), b.astype(np.uint64))
    q = ua // ub
    neg = (a < 0) != (b < 0)
    return np.where(neg, (-q), q).astype(np.int64)


def _eval(node, ctx):
    t = type(node).__name__
    kind = ctx["kind"]
    dt = _DT[kind]
    if t == "Num":
        v = int(node.value) if kind == "int64" else float(node.value)
        return np.full(ctx["shape"], v, dtype=dt)
    if t == "Param":
        v = ctx["params"][node.name]
        v = int(v) if kind == "int64" else float(v)
        return np.full(ctx["shape"], v, dtype=dt)
    if t == "IdComponent":
        return ctx["ids"][node.axis].astype(dt)
    if t == "Read":
        acc = ctx["accs"][node.accessor]
        src = ctx["views"][node.accessor]
        ext = src.shape
        idx = []
        for j, off in enumerate(node.offsets):
            idx.append(np.clip(ctx["ids"][j] + off, 0, ext[j] - 1))
        idx = tuple(idx)
        ok = ctx["masks"][node.accessor][idx]
        if not np.all(ok):
            raise OracleError("mapper", f"accessor '{acc.name}' read outside its mapped region")
        return src[idx].astype(dt)
    if t == "Neg":
        with np.errstate(all="ignore"):
            return (-_eval(node.operand, ctx)).astype(dt)
    if t == "BinOp":
        a = _eval(node.left, ctx)
        b = _eval(node.right, ctx)
        with np.errstate(all="ignore"):
            if node.op == "+":
                r = a + b
            elif node.op == "-":
                r = a - b
            elif node.op == "*":
                r = a * b
            elif kind == "int64":
                r = _wrap_div(a, b)
            else:
                r = a / b
        return r.astype(dt)
    raise TypeError(t)


def run_serial(buffers, tasks):
    """Final buffer contents of the program (node_count = 1 semantics)."""
    arrays = {name: initial_array(b) for name, b in buffers.items()}
    for task in tasks:
        if not isinstance(task.body, dict):
            raise TypeError("native bodies have their own oracles (oracle.native)")
        lo, hi = task.global_range.mins, task.global_range.maxs
        shape = tuple(b - a for a, b in zip(lo, hi))
        ids = np.meshgrid(*[np.arange(a, b, dtype=np.int64) for a, b in zip(lo, hi)], indexing="ij")
        accs = {a.name: a for a in task.accessors}
        views, masks = {}, {}
        for a in task.accessors:
            if a.mode.value == "read":
                views[a.name] = arrays[a.buffer].copy()  # pre-task snapshot
                masks[a.name] = _mapped_mask(a.mapper, lo, hi, arrays[a.buffer].shape)
        results = {}
        for a in task.accessors:
            if a.mode.value != "write":
                continue
            kind = buffers[a.buffer].element_kind
            ctx = {"kind": kind, "shape": shape, "ids": ids, "params": task.params,
                   "accs": accs, "views": views, "masks": masks}
            results[a.buffer] = _eval(task.body[a.name], ctx)
        for buf, vals in results.items():
            sl = tuple(slice(a, b) for a, b in zip(lo, hi))
            arrays[buf][sl] = vals
    return arrays


def same_bits(a, b) -> bool:
    """Bitwise equality, NaN == NaN regardless of payload/sign."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind == "f":
        na, nb = np.isnan(a), np.isnan(b)
        if not np.array_equal(na, nb):
            return False
        iv = np.int64 if a.itemsize == 8 else np.int32
        return np.array_equal(np.where(na, 0, a).view(iv), np.where(nb, 0, b).view(iv))
    return np.array_equal(a, b)
