"""The task-body expression language: AST, parser, printer and lowering.

Grammar and semantics are the reference's (pkg/src/clusterq/kernel.py:3-19):

    expr   := term (('+' | '-') term)*
    term   := unary (('*' | '/') unary)*
    unary  := '-'? factor
    factor := number | param | id_component | access | '(' expr ')'
    access := name '[' index (',' index)* ']'
    index  := 'i' '.' digit (('+' | '-') integer)?

Bare ``i`` means ``i.0`` in a 1-D kernel.  Errors carry the same types and
character positions as the reference parser (kernel.py:68-213) so scenario
diagnostics stay identical.

Evaluation does NOT happen on the host here.  ``lower()`` turns a body into a
postfix program (``Program``) that the sm_100a expression kernel
(csrc/cq_kernels.cu, ``cq_expr_eval``) interprets per cell with the
reference's numeric rules: IEEE binary64 with one rounding per operator, or
wrapping int64 with truncating division (kernel.py:275-331), or -- for the
new ``float32`` element kind -- binary32 with one rounding per operator.
Bodies that match a recognised pattern (SAXPY, the 2-D 5-point wave step)
are additionally routed to hand-written kernels with the same operator order.
"""

import re
from dataclasses import dataclass
from typing import Union

from .errors import KernelNameError, KernelSyntaxError, ValidationError


@dataclass(frozen=True)
class Num:
    value: Union[int, float]


@dataclass(frozen=True)
class Param:
    name: str


@dataclass(frozen=True)
class IdComponent:
    axis: int


@dataclass(frozen=True)
class Read:
    accessor: str
    offsets: tuple


@dataclass(frozen=True)
class Neg:
    operand: "Expr"


@dataclass(frozen=True)
class BinOp:
    op: str
    left: "Expr"
    right: "Expr"


Expr = Union[Num, Param, IdComponent, Read, Neg, BinOp]

_NUM_RE = re.compile(r"\d+\.\d*(?:[eE][+-]?\d+)?|\d+[eE][+-]?\d+|\d+")
_IDENT_RE = re.compile(r"[A-Za-z_]\w*")
_INT_RE = re.compile(r"\d+")


class _Cursor:
    """Character cursor over kernel text with whitespace skipping."""

    __slots__ = ("src", "at", "arity", "params", "dims")

    def __init__(self, src, arity, params, dims):
        self.src = src
        self.at = 0
        self.arity = dict(arity)
        self.params = set(params)
        self.dims = dims

    def look(self):
        """Next significant character ('' at the end); skips whitespace."""
        n = len(self.src)
        while self.at < n and self.src[self.at].isspace():
            self.at += 1
        return self.src[self.at] if self.at < n else ""

    def take(self, ch):
        got = self.look()
        if got != ch:
            raise KernelSyntaxError(f"expected {ch!r}, got {(got or 'end of input')!r}", self.at)
        self.at += 1


def _parse_sum(c):
    node = _parse_product(c)
    while True:
        ch = c.look()
        if ch != "+" and ch != "-":
            return node
        c.at += 1
        node = BinOp(ch, node, _parse_product(c))


def _parse_product(c):
    node = _parse_signed(c)
    while True:
        ch = c.look()
        if ch != "*" and ch != "/":
            return node
        c.at += 1
        node = BinOp(ch, node, _parse_signed(c))


def _parse_signed(c):
    if c.look() == "-":
        c.at += 1
        return Neg(_parse_atom(c))
    return _parse_atom(c)


def _parse_atom(c):
    ch = c.look()
    if ch == "(":
        c.at += 1
        inner = _parse_sum(c)
        c.take(")")
        return inner
    if ch.isdigit():
        m = _NUM_RE.match(c.src, c.at)
        if m is None:
            raise KernelSyntaxError("malformed number", c.at)
        c.at = m.end()
        text = m.group(0)
        is_float = any(k in text for k in ".eE")
        return Num(float(text) if is_float else int(text))
    m = _IDENT_RE.match(c.src, c.at)
    if m is None:
        raise KernelSyntaxError(f"expected a value, got {(ch or 'end of input')!r}", c.at)
    word, begin = m.group(0), c.at
    c.at = m.end()
    if word == "i":
        return IdComponent(_parse_axis(c, begin))
    if c.look() == "[":
        return _parse_access(c, word, begin)
    if word in c.params:
        return Param(word)
    if word in c.arity:
        raise KernelNameError(f"accessor '{word}' must be indexed, e.g. {word}[i.0]")
    raise KernelNameError(f"unknown name '{word}'")


def _parse_axis(c, begin):
    """Axis of an id component whose 'i' is already consumed."""
    if c.look() != ".":
        if c.dims != 1:
            raise KernelSyntaxError("bare 'i' is only valid in 1D; use i.<axis>", begin)
        return 0
    c.at += 1
    ch = c.look()
    if not ch.isdigit():
        raise KernelSyntaxError("expected an axis digit after 'i.'", c.at)
    c.at += 1
    axis = int(ch)
    if axis >= c.dims:
        raise KernelSyntaxError(f"id component i.{axis} out of range for a {c.dims}D kernel", begin)
    return axis


def _parse_access(c, name, begin):
    if name not in c.arity:
        raise KernelNameError(f"unknown accessor '{name}'")
    c.take("[")
    offsets = []
    while True:
        offsets.append(_parse_index(c, len(offsets)))
        if c.look() == ",":
            c.at += 1
            continue
        c.take("]")
        break
    want = c.arity[name]
    if len(offsets) != want:
        raise KernelSyntaxError(f"accessor '{name}' takes {want} indices, got {len(offsets)}", begin)
    return Read(name, tuple(offsets))


def _parse_index(c, slot):
    m = _IDENT_RE.match(c.src, c.at) if c.look() else None
    if m is None or m.group(0) != "i":
        if m is not None:
            raise KernelNameError(f"unknown name '{m.group(0)}' in index")
        raise KernelSyntaxError(f"expected an id component, got {(c.look() or 'end of input')!r}", c.at)
    begin = c.at
    c.at = m.end()
    axis = _parse_axis(c, begin)
    if axis != slot:
        raise KernelSyntaxError(f"index {slot} must use i.{slot}", begin)
    sign = c.look()
    if sign != "+" and sign != "-":
        return 0
    c.at += 1
    c.look()
    m = _INT_RE.match(c.src, c.at)
    if m is None:
        raise KernelSyntaxError("accessor offset must be a constant integer", c.at)
    c.at = m.end()
    return int(m.group(0)) * (1 if sign == "+" else -1)


def parse_kernel(text, reads, params, dims) -> Expr:
    """Parse ``text``; ``reads`` maps accessor name to index arity, ``params``
    is the set of scalar parameter names, ``dims`` the kernel dimensionality."""
    c = _Cursor(text, reads, params, dims)
    tree = _parse_sum(c)
    c.look()
    if c.at != len(c.src):
        raise KernelSyntaxError(f"unexpected {c.src[c.at]!r}", c.at)
    return tree


# ----------------------------------------------------------------- printing

_BIN_RANK = {"+": 1, "-": 1, "*": 2, "/": 2}


def _rank(e) -> int:
    if isinstance(e, BinOp):
        return _BIN_RANK[e.op]
    return 3 if isinstance(e, Neg) else 4


def format_kernel(expr) -> str:
    """Canonical text; reparsing it reproduces the same tree."""
    if isinstance(expr, Num):
        return repr(expr.value)
    if isinstance(expr, Param):
        return expr.name
    if isinstance(expr, IdComponent):
        return f"i.{expr.axis}"
    if isinstance(expr, Read):
        parts = []
        for axis, off in enumerate(expr.offsets):
            parts.append(f"i.{axis}" if off == 0 else f"i.{axis}{off:+d}")
        return f"{expr.accessor}[{', '.join(parts)}]"
    if isinstance(expr, Neg):
        inner = format_kernel(expr.operand)
        return f"-({inner})" if _rank(expr.operand) < 4 else f"-{inner}"
    if isinstance(expr, BinOp):
        r = _BIN_RANK[expr.op]
        lhs = format_kernel(expr.left)
        rhs = format_kernel(expr.right)
        if _rank(expr.left) < r:
            lhs = f"({lhs})"
        if _rank(expr.right) <= r:
            rhs = f"({rhs})"
        return f"{lhs} {expr.op} {rhs}"
    raise TypeError(f"not a kernel expression: {expr!r}")


def walk(expr):
    """Pre-order, depth-first traversal of every node."""
    stack = [expr]
    while stack:
        node = stack.pop()
        yield node
        if isinstance(node, BinOp):
            stack.append(node.right)
            stack.append(node.left)
        elif isinstance(node, Neg):
            stack.append(node.operand)


_I64_MOD = 1 << 64
_I64_MIN = -(1 << 63)
_I64_MAX = (1 << 63) - 1


def wrap_i64(v: int) -> int:
    """Two's-complement wrap of an arbitrary Python int to int64."""
    v %= _I64_MOD
    return v - _I64_MOD if v > _I64_MAX else v


# ---------------------------------------------------------------- lowering

# Opcodes of the device expression interpreter (keep in sync with
# csrc/cq_kernels.cu: enum CqOp).
OP_CONST = 0   # push consts[arg]
OP_ID = 1      # push global id component arg
OP_READ = 2    # push read slot arg (slot table holds accessor + offsets)
OP_NEG = 3
OP_ADD = 4
OP_SUB = 5
OP_MUL = 6
OP_DIV = 7

_BIN_CODE = {"+": OP_ADD, "-": OP_SUB, "*": OP_MUL, "/": OP_DIV}


@dataclass(frozen=True)
class Program:
    """Postfix form of one body expression for the device interpreter.

    ``code`` is a flat tuple of (opcode, argument) pairs; ``consts`` holds
    literal/parameter values already converted to the evaluation kind (the
    host performs ``float(v)`` / ``int(v)`` exactly as the reference does at
    every use, kernel.py:293-299); ``reads`` lists (accessor, offsets) per
    read slot; ``depth`` is the maximum stack depth.
    """

    code: tuple
    consts: tuple
    reads: tuple
    depth: int


MAX_STACK = 32
MAX_CODE = 256
MAX_READ_SLOTS = 32


def lower(expr, params, kind) -> Program:
    """Lower an expression to a ``Program`` for element kind ``kind``
    ("float64", "float32" or "int64")."""
    integer = kind == "int64"
    code = []
    consts = []
    slots = []
    slot_of = {}
    depth = 0
    peak = 0

    def const(v):
        if integer:
            iv = int(v)
            if not _I64_MIN <= iv <= _I64_MAX:
                # The reference would carry an unbounded Python int into the
                # operator; the device is 64-bit only.
                raise ValidationError(f"integer constant {iv} does not fit in int64")
            consts.append(iv)
        else:
            consts.append(float(v))
        return len(consts) - 1

    def emit(node):
        nonlocal depth, peak
        if isinstance(node, Num):
            code.append((OP_CONST, const(node.value)))
            depth += 1
        elif isinstance(node, Param):
            code.append((OP_CONST, const(params[node.name])))
            depth += 1
        elif isinstance(node, IdComponent):
            code.append((OP_ID, node.axis))
            depth += 1
        elif isinstance(node, Read):
            key = (node.accessor, tuple(node.offsets))
            if key not in slot_of:
                slot_of[key] = len(slots)
                slots.append(key)
            code.append((OP_READ, slot_of[key]))
            depth += 1
        elif isinstance(node, Neg):
            emit(node.operand)
            code.append((OP_NEG, 0))
        elif isinstance(node, BinOp):
            emit(node.left)
            emit(node.right)
            code.append((_BIN_CODE[node.op], 0))
            depth -= 1
        else:
            raise TypeError(f"not a kernel expression: {node!r}")
        peak = max(peak, depth)

    emit(expr)
    if peak > MAX_STACK:
        raise ValidationError(f"expression needs stack depth {peak} > {MAX_STACK}")
    if len(code) > MAX_CODE:
        raise ValidationError(f"expression has {len(code)} operations > {MAX_CODE}")
    if len(slots) > MAX_READ_SLOTS:
        raise ValidationError(f"expression has {len(slots)} distinct reads > {MAX_READ_SLOTS}")
    return Program(tuple(code), tuple(consts), tuple(slots), peak)
