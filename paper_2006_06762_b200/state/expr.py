"""Scalar expression language of compute bodies (host-side data model).

Mirror of the reference's expression types (`src/expr.py:33-188`): the GPU
runner, the State encoder and the feature kernel read these objects, and the
reference's own objects have the same class names and fields, so either can be
handed to this package.  Only the structural parts the hot path needs live
here: affine index forms, node types, walks, op counting
(`src/expr.py:303-331`), inlining substitution (`src/expr.py:224-268`) and the
JSON codec (`src/expr.py:404-447`).  Numeric evaluation is not here: values
are computed by generated CUDA (see `codegen.py`), and the CPU evaluator used
to check them lives under `oracle/`.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator


@dataclass(frozen=True)
class Lin:
    """sum(coeff * iterator) + const, terms sorted by iterator name."""

    terms: tuple = ()
    const: int = 0

    @staticmethod
    def var(name: str, coeff: int = 1) -> "Lin":
        return Lin(((name, coeff),), 0) if coeff else Lin((), 0)

    @staticmethod
    def of(const: int) -> "Lin":
        return Lin((), const)

    def __add__(self, other: "Lin") -> "Lin":
        merged: dict = {}
        for name, c in self.terms + other.terms:
            merged[name] = merged.get(name, 0) + c
        return Lin(tuple(sorted((n, c) for n, c in merged.items() if c)),
                   self.const + other.const)

    def shift(self, k: int) -> "Lin":
        return Lin(self.terms, self.const + k)

    def scale(self, k: int) -> "Lin":
        if k == 0:
            return Lin((), 0)
        return Lin(tuple((n, c * k) for n, c in self.terms), self.const * k)

    def iters(self) -> frozenset:
        return frozenset(n for n, _ in self.terms)

    def coeff(self, name: str) -> int:
        return dict(self.terms).get(name, 0)

    def is_single_var(self) -> bool:
        return self.const == 0 and len(self.terms) == 1 and self.terms[0][1] == 1

    def substitute(self, mapping: dict) -> "Lin":
        out = Lin.of(self.const)
        for name, c in self.terms:
            out = out + mapping.get(name, Lin.var(name)).scale(c)
        return out

    def interval(self, ranges: dict) -> tuple:
        lo = hi = self.const
        for name, c in self.terms:
            a, b = ranges[name]
            lo, hi = (lo + c * a, hi + c * b) if c >= 0 else (lo + c * b, hi + c * a)
        return lo, hi


BINARY_OPS = ("add", "sub", "mul", "div", "max", "min", "lt", "le", "gt", "ge", "eq")
COMPARE_OPS = ("lt", "le", "gt", "ge", "eq")
CALL_FNS = ("exp", "sqrt", "log", "abs")
REDUCE_OPS = ("sum", "max")


@dataclass(frozen=True)
class Const:
    value: float


@dataclass(frozen=True)
class IterVal:
    lin: Lin


@dataclass(frozen=True)
class Read:
    buffer: str
    index: tuple


@dataclass(frozen=True)
class Bin:
    op: str
    lhs: object
    rhs: object

    def __post_init__(self) -> None:
        if self.op not in BINARY_OPS:
            raise ValueError(f"unknown binary op {self.op!r}")


@dataclass(frozen=True)
class Call:
    fn: str
    arg: object

    def __post_init__(self) -> None:
        if self.fn not in CALL_FNS:
            raise ValueError(f"unknown call {self.fn!r}")


@dataclass(frozen=True)
class Select:
    cond: object
    then: object
    other: object


@dataclass(frozen=True)
class Reduce:
    op: str
    axes: tuple
    body: object

    def __post_init__(self) -> None:
        if self.op not in REDUCE_OPS:
            raise ValueError(f"unknown reduce op {self.op!r}")


def kind(e) -> str:
    """Class name dispatch, so reference objects work here too."""
    return type(e).__name__


def children(e) -> tuple:
    k = kind(e)
    if k == "Bin":
        return (e.lhs, e.rhs)
    if k == "Call":
        return (e.arg,)
    if k == "Select":
        return (e.cond, e.then, e.other)
    if k == "Reduce":
        return (e.body,)
    return ()


def walk(e) -> Iterator:
    """Pre-order walk (the order `reads` and `op_counts` depend on)."""
    stack = [e]
    while stack:
        n = stack.pop()
        yield n
        stack.extend(reversed(children(n)))


def reads(e) -> tuple:
    return tuple(n for n in walk(e) if kind(n) == "Read")


def iter_names(e) -> frozenset:
    out: set = set()
    for n in walk(e):
        k = kind(n)
        if k == "IterVal":
            out |= set(n.lin.iters())
        elif k == "Read":
            for lin in n.index:
                out |= set(lin.iters())
        elif k == "Reduce":
            out |= set(n.axes)
    return frozenset(out)


def validate_expr(e, at_root: bool = True) -> list:
    out = []
    if kind(e) == "Reduce":
        if not at_root:
            out.append("reduction below expression root")
        return out + validate_expr(e.body, False)
    for c in children(e):
        out += validate_expr(c, False)
    return out


OP_KIND = {"add": "add", "sub": "sub", "mul": "mul", "div": "div",
           "max": "minmax", "min": "minmax",
           "lt": "cmp", "le": "cmp", "gt": "cmp", "ge": "cmp", "eq": "cmp"}


def op_counts(e) -> dict:
    """Per-point float op counts by kind (`src/expr.py:303-327`)."""
    acc: dict = {}
    for n in walk(e):
        k = kind(n)
        if k == "Bin":
            b = OP_KIND[n.op]
        elif k == "Call":
            b = "math_call"
        elif k == "Select":
            b = "select"
        elif k == "Reduce":
            b = "add" if n.op == "sum" else "minmax"
        else:
            continue
        acc[b] = acc.get(b, 0) + 1
    return acc


def ops_per_point(e) -> int:
    return sum(op_counts(e).values())


def substitute_iters(e, mapping: dict):
    k = kind(e)
    if k == "Const":
        return e
    if k == "IterVal":
        return IterVal(e.lin.substitute(mapping))
    if k == "Read":
        return Read(e.buffer, tuple(l.substitute(mapping) for l in e.index))
    if k == "Bin":
        return Bin(e.op, substitute_iters(e.lhs, mapping), substitute_iters(e.rhs, mapping))
    if k == "Call":
        return Call(e.fn, substitute_iters(e.arg, mapping))
    if k == "Select":
        return Select(*(substitute_iters(x, mapping) for x in (e.cond, e.then, e.other)))
    if k == "Reduce":
        hit = set(e.axes) & set(mapping)
        if hit:
            raise ValueError(f"substitution touches reduction axes {sorted(hit)}")
        return Reduce(e.op, e.axes, substitute_iters(e.body, mapping))
    raise TypeError(f"not an expression: {e!r}")


def inline_reads(e, buffer: str, space: tuple, body):
    """Replace reads of `buffer` by the producer body composed on the read index."""
    k = kind(e)
    if k == "Read" and e.buffer == buffer:
        if len(e.index) != len(space):
            raise ValueError(f"read of {buffer} has rank {len(e.index)}, expected {len(space)}")
        return substitute_iters(body, dict(zip(space, e.index)))
    if k in ("Const", "IterVal", "Read"):
        return e
    if k == "Bin":
        return Bin(e.op, inline_reads(e.lhs, buffer, space, body),
                   inline_reads(e.rhs, buffer, space, body))
    if k == "Call":
        return Call(e.fn, inline_reads(e.arg, buffer, space, body))
    if k == "Select":
        return Select(*(inline_reads(x, buffer, space, body) for x in (e.cond, e.then, e.other)))
    if k == "Reduce":
        return Reduce(e.op, e.axes, inline_reads(e.body, buffer, space, body))
    raise TypeError(f"not an expression: {e!r}")


# ---------------------------------------------------------------------------
# JSON codec (same wire format as `src/expr.py:404-447`)
# ---------------------------------------------------------------------------


def lin_to_json(l) -> dict:
    return {"t": [[n, c] for n, c in l.terms], "c": l.const}


def lin_from_json(d: dict) -> Lin:
    return Lin(tuple((str(n), int(c)) for n, c in d["t"]), int(d["c"]))


def expr_to_json(e) -> dict:
    k = kind(e)
    if k == "Const":
        return {"k": "const", "v": e.value}
    if k == "IterVal":
        return {"k": "iter", "lin": lin_to_json(e.lin)}
    if k == "Read":
        return {"k": "read", "buf": e.buffer, "idx": [lin_to_json(l) for l in e.index]}
    if k == "Bin":
        return {"k": "bin", "op": e.op, "a": expr_to_json(e.lhs), "b": expr_to_json(e.rhs)}
    if k == "Call":
        return {"k": "call", "fn": e.fn, "a": expr_to_json(e.arg)}
    if k == "Select":
        return {"k": "select", "c": expr_to_json(e.cond), "t": expr_to_json(e.then),
                "o": expr_to_json(e.other)}
    if k == "Reduce":
        return {"k": "reduce", "op": e.op, "axes": list(e.axes), "body": expr_to_json(e.body)}
    raise TypeError(f"not an expression: {e!r}")


def expr_from_json(d: dict):
    k = d["k"]
    if k == "const":
        return Const(float(d["v"]))
    if k == "iter":
        return IterVal(lin_from_json(d["lin"]))
    if k == "read":
        return Read(str(d["buf"]), tuple(lin_from_json(x) for x in d["idx"]))
    if k == "bin":
        return Bin(str(d["op"]), expr_from_json(d["a"]), expr_from_json(d["b"]))
    if k == "call":
        return Call(str(d["fn"]), expr_from_json(d["a"]))
    if k == "select":
        return Select(expr_from_json(d["c"]), expr_from_json(d["t"]), expr_from_json(d["o"]))
    if k == "reduce":
        return Reduce(str(d["op"]), tuple(str(a) for a in d["axes"]), expr_from_json(d["body"]))
    raise ValueError(f"unknown expression tag {k!r}")
