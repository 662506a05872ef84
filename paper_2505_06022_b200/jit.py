"""DSL -> CUDA JIT.

A task body's postfix program (kernel.lower) is turned into straight-line
CUDA C++ -- one rounding intrinsic per DSL operator, in the tree's order,
reads clamped per buffer axis like ReadView.read (model.py:442-446) -- and
compiled once per program *shape* with NVRTC for sm_100a (csrc/cq_jit.cu).
The kernel consumes the same ``cq_expr_t`` block as the device interpreter,
so constants, parameters, views and the box are runtime data: the 100 tasks
of a wave program share one compiled kernel.  Results are bit-identical to
the interpreter (tests/test_gpu_parity.py checks every golden program on
both).  Bodies that need the per-cell mapper check stay on the interpreter.
"""

import ctypes
import hashlib
import os

from . import _native as N
from .kernel import OP_ADD, OP_CONST, OP_DIV, OP_ID, OP_MUL, OP_NEG, OP_READ, OP_SUB

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(HERE), "include", "cq.h")

# "auto": JIT for launches of at least this many cells; "1" always; "0" never
MODE = os.environ.get("CQ_JIT", "auto")
AUTO_MIN_CELLS = 1 << 16

_STDINT = """
typedef signed char int8_t; typedef short int16_t; typedef int int32_t; typedef long long int64_t;
typedef unsigned char uint8_t; typedef unsigned short uint16_t; typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
"""

_OPS = {
    0: ("double", "__dadd_rn({a}, {b})", "__dsub_rn({a}, {b})", "__dmul_rn({a}, {b})",
        "__ddiv_rn({a}, {b})", "(-{a})", "__longlong_as_double(X.consts[{i}])", "((double){p})"),
    1: ("float", "__fadd_rn({a}, {b})", "__fsub_rn({a}, {b})", "__fmul_rn({a}, {b})",
        "__fdiv_rn({a}, {b})", "(-{a})", "__double2float_rn(__longlong_as_double(X.consts[{i}]))",
        "__ll2float_rn({p})"),
    2: ("long long", "(long long)((unsigned long long){a} + (unsigned long long){b})",
        "(long long)((unsigned long long){a} - (unsigned long long){b})",
        "(long long)((unsigned long long){a} * (unsigned long long){b})", None,
        "(long long)(0ull - (unsigned long long){a})", "X.consts[{i}]", "((long long){p})"),
}

_cache = {}
_headers = None


def enabled_for(cells: int) -> bool:
    if MODE == "0":
        return False
    return MODE == "1" or cells >= AUTO_MIN_CELLS


def _header_blobs():
    global _headers
    if _headers is None:
        with open(HEADER) as fh:
            _headers = (fh.read(), _STDINT)
    return _headers


def generate(kind: int, kdims: int, outs, slots, view_dims):
    """CUDA source for one program shape.

    outs: [(code list of (op, arg)), ...] per output (args already remapped
    to the packed block: const index, padded axis, slot index);
    slots: [(view index, offsets)]; view_dims: dims per view index."""
    T, add, sub, mul, div, neg, const, idc = _OPS[kind]
    lines = [
        '#include "cq.h"',
        "extern \"C\" __global__ void __launch_bounds__(256) KERNEL(const __grid_constant__ cq_expr_t X,",
        "                                                         unsigned long long* flag) {",
        "  const long long n1 = X.box.hi[1] - X.box.lo[1], n2 = X.box.hi[2] - X.box.lo[2];",
        "  const long long total = (X.box.hi[0] - X.box.lo[0]) * n1 * n2;",
        "  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;",
        "       t += (long long)gridDim.x * blockDim.x) {",
        "    const long long p2 = X.box.lo[2] + t % n2, r_ = t / n2;",
        "    const long long p1 = X.box.lo[1] + r_ % n1, p0 = X.box.lo[0] + r_ / n1;",
        "    const long long p[3] = {p0, p1, p2};",
        "    bool failed = false;",
    ]
    for s, (vi, offs) in enumerate(slots):
        bd = view_dims[vi]
        q = ["0", "0", "0"]
        for j, off in enumerate(offs):
            ax = 3 - bd + j
            src = f"p[{3 - kdims + j}] + ({off})"
            q[ax] = (f"min(max({src}, X.view_extent[{vi}].lo[{ax}]), "
                     f"X.view_extent[{vi}].hi[{ax}] - 1)")
        lines.append(f"    const long long q{s}_0 = {q[0]}, q{s}_1 = {q[1]}, q{s}_2 = {q[2]};")
        lines.append(f"    const {T} r{s} = ((const {T}*)X.views[{vi}].ptr)[(q{s}_0 - X.views[{vi}].alloc.lo[0]) * "
                     f"X.views[{vi}].stride[0] + (q{s}_1 - X.views[{vi}].alloc.lo[1]) * X.views[{vi}].stride[1] + "
                     f"(q{s}_2 - X.views[{vi}].alloc.lo[2]) * X.views[{vi}].stride[2]];")
    tmp = 0
    results = []
    for code in outs:
        stack = []
        for op, arg in code:
            name = f"v{tmp}"
            tmp += 1
            if op == OP_CONST:
                expr = const.format(i=arg)
            elif op == OP_ID:
                expr = idc.format(p=f"p[{arg}]")
            elif op == OP_READ:
                expr = f"r{arg}"
            elif op == OP_NEG:
                expr = neg.format(a=stack.pop())
            else:
                b = stack.pop()
                a = stack.pop()
                if op == OP_ADD:
                    expr = add.format(a=a, b=b)
                elif op == OP_SUB:
                    expr = sub.format(a=a, b=b)
                elif op == OP_MUL:
                    expr = mul.format(a=a, b=b)
                elif kind != 2:
                    expr = div.format(a=a, b=b)
                else:
                    lines.append(f"    long long {name};")
                    lines.append(f"    if ({b} == 0) {{ failed = true; {name} = 0;"
                                 f" unsigned long long key = ((unsigned long long)t << 4) | 7ull;"
                                 f" unsigned long long old = atomicMin(flag, key);"
                                 f" if (old > key) {{ long long* pt = (long long*)(flag + 1);"
                                 f" pt[0] = p0; pt[1] = p1; pt[2] = p2; }} }}")
                    lines.append(f"    else {{ unsigned long long ua = {a} < 0 ? 0ull - (unsigned long long){a}"
                                 f" : (unsigned long long){a}; unsigned long long ub = {b} < 0 ?"
                                 f" 0ull - (unsigned long long){b} : (unsigned long long){b};"
                                 f" unsigned long long uq = ua / ub;"
                                 f" {name} = (long long)((({a} < 0) != ({b} < 0)) ? 0ull - uq : uq); }}")
                    stack.append(name)
                    continue
            lines.append(f"    const {T} {name} = {expr};")
            stack.append(name)
        results.append(stack[-1])
    lines.append("    if (failed) continue;")
    for o, res in enumerate(results):
        lines.append(f"    (({T}*)X.out[{o}].ptr)[(p0 - X.out[{o}].alloc.lo[0]) * X.out[{o}].stride[0] + "
                     f"(p1 - X.out[{o}].alloc.lo[1]) * X.out[{o}].stride[1] + "
                     f"(p2 - X.out[{o}].alloc.lo[2]) * X.out[{o}].stride[2]] = {res};")
    lines += ["  }", "}"]
    body = "\n".join(lines)
    digest = hashlib.sha1(body.encode()).hexdigest()[:16]
    name = f"cq_jit_{digest}"
    return name, body.replace("KERNEL", name)


def handle_for(kind, kdims, outs, slots, view_dims) -> int:
    """Compiled kernel handle (NVRTC once per program shape per process)."""
    name, src = generate(kind, kdims, outs, slots, view_dims)
    h = _cache.get(src)
    if h is None:
        hdr, stdint = _header_blobs()
        srcs = (ctypes.c_char_p * 2)(hdr.encode(), stdint.encode())
        names = (ctypes.c_char_p * 2)(b"cq.h", b"stdint.h")
        out = ctypes.c_uint64()
        N.call("cq_jit_compile", src.encode(), name.encode(), 2, srcs, names, ctypes.byref(out))
        h = _cache[src] = out.value
    return h
