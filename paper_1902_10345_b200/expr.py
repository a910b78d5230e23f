"""Symbolic expressions of the SDFG interchange text, re-parsed host-side.

The reference serialises every expression, range and subset as grammar text
(serialization.py:54-71; grammar in symbolic.py:1-12): integer arithmetic
``+ - * // %``, ``min``/``max``, comparisons and boolean connectives; ranges
are inclusive ``begin:end[:stride[:tilesize]]`` (symbolic.py:579-660); a
subset is ``[r0, r1, ...]`` (symbolic.py:669-727).  The grammar is a subset
of Python expression syntax, so it is parsed with :mod:`ast` into a small
tree.  ``//`` and ``%`` follow floor semantics exactly like the reference's
``sdfg_fdiv``/``sdfg_fmod`` (tasklets.py:336-347).

Besides evaluation, :func:`affine` decomposes index expressions into
``{symbol: coeff} + const`` -- the form the motif classifier reasons in.
"""

from __future__ import annotations

import ast
from dataclasses import dataclass
from typing import Mapping, Optional, Union

Number = Union[int, float]


class ExprError(ValueError):
    pass


@dataclass(frozen=True)
class Expr:
    pass


@dataclass(frozen=True)
class Num(Expr):
    value: Number

    def __str__(self):
        return repr(self.value)


@dataclass(frozen=True)
class Sym(Expr):
    name: str

    def __str__(self):
        return self.name


@dataclass(frozen=True)
class Bin(Expr):
    op: str  # + - * // % /
    left: Expr
    right: Expr

    def __str__(self):
        return f"({self.left} {self.op} {self.right})"


@dataclass(frozen=True)
class Neg(Expr):
    arg: Expr

    def __str__(self):
        return f"(-{self.arg})"


@dataclass(frozen=True)
class Call(Expr):
    fn: str  # min | max | size
    args: tuple

    def __str__(self):
        return f"{self.fn}({', '.join(map(str, self.args))})"


@dataclass(frozen=True)
class Cmp(Expr):
    op: str
    left: Expr
    right: Expr

    def __str__(self):
        return f"({self.left} {self.op} {self.right})"


@dataclass(frozen=True)
class BoolOp(Expr):
    op: str  # and | or
    args: tuple


@dataclass(frozen=True)
class Not(Expr):
    arg: Expr


_BIN = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*", ast.FloorDiv: "//", ast.Mod: "%",
        ast.Div: "/"}
_CMP = {ast.Lt: "<", ast.LtE: "<=", ast.Gt: ">", ast.GtE: ">=", ast.Eq: "==",
        ast.NotEq: "!="}


def _conv(node: ast.AST) -> Expr:
    if isinstance(node, ast.Expression):
        return _conv(node.body)
    if isinstance(node, ast.Constant) and isinstance(node.value, (int, float)) \
            and not isinstance(node.value, bool):
        return Num(node.value)
    if isinstance(node, ast.Constant) and isinstance(node.value, bool):
        return Num(int(node.value))
    if isinstance(node, ast.Name):
        return Sym(node.id)
    if isinstance(node, ast.BinOp) and type(node.op) in _BIN:
        return Bin(_BIN[type(node.op)], _conv(node.left), _conv(node.right))
    if isinstance(node, ast.UnaryOp):
        if isinstance(node.op, ast.USub):
            inner = _conv(node.operand)
            if isinstance(inner, Num):
                return Num(-inner.value)
            return Neg(inner)
        if isinstance(node.op, ast.UAdd):
            return _conv(node.operand)
        if isinstance(node.op, ast.Not):
            return Not(_conv(node.operand))
    if isinstance(node, ast.Call) and isinstance(node.func, ast.Name) \
            and node.func.id in ("min", "max", "size") and not node.keywords:
        return Call(node.func.id, tuple(_conv(a) for a in node.args))
    if isinstance(node, ast.Compare) and len(node.ops) == 1 and type(node.ops[0]) in _CMP:
        return Cmp(_CMP[type(node.ops[0])], _conv(node.left), _conv(node.comparators[0]))
    if isinstance(node, ast.BoolOp):
        return BoolOp("and" if isinstance(node.op, ast.And) else "or",
                      tuple(_conv(v) for v in node.values))
    raise ExprError(f"unsupported expression syntax: {ast.dump(node)}")


def parse_expr(text: str) -> Expr:
    try:
        tree = ast.parse(text.strip(), mode="eval")
    except SyntaxError as exc:
        raise ExprError(f"cannot parse expression {text!r}: {exc}") from exc
    return _conv(tree)


def _split_top(text: str, sep: str) -> list[str]:
    """Split on ``sep`` outside parentheses/brackets (symbolic.py:621-633)."""
    parts, depth, start = [], 0, 0
    for i, c in enumerate(text):
        if c in "([":
            depth += 1
        elif c in ")]":
            depth -= 1
        elif c == sep and depth == 0:
            parts.append(text[start:i])
            start = i + 1
    parts.append(text[start:])
    return parts


@dataclass(frozen=True)
class Range:
    """Inclusive begin:end:stride:tilesize (symbolic.py:579-618)."""
    begin: Expr
    end: Expr
    stride: Expr = Num(1)
    tile: Expr = Num(1)

    @property
    def is_point(self) -> bool:
        return self.begin == self.end and self.stride == Num(1) and self.tile == Num(1)

    def __str__(self):
        if self.is_point:
            return str(self.begin)
        return f"{self.begin}:{self.end}" + ("" if self.stride == Num(1) and self.tile == Num(1)
                                             else f":{self.stride}")


def parse_range(text: str) -> Range:
    parts = [p.strip() for p in _split_top(text, ":")]
    if not 1 <= len(parts) <= 4 or any(p == "" for p in parts):
        raise ExprError(f"bad range {text!r}")
    ex = [parse_expr(p) for p in parts]
    if len(ex) == 1:
        return Range(ex[0], ex[0])
    return Range(*ex)


def parse_subset(text: str) -> tuple[Range, ...]:
    t = text.strip()
    if not (t.startswith("[") and t.endswith("]")):
        raise ExprError(f"bad subset {text!r}")
    return tuple(parse_range(p) for p in _split_top(t[1:-1], ","))


# ---------------------------------------------------------------- evaluation

def _fdiv(a, b):
    if isinstance(a, float) or isinstance(b, float):
        import math
        return math.floor(a / b)
    return a // b  # Python floor semantics == sdfg_fdiv


def evaluate(e: Expr, env: Mapping[str, Number]) -> Number:
    if isinstance(e, Num):
        return e.value
    if isinstance(e, Sym):
        if e.name not in env:
            raise ExprError(f"unbound symbol '{e.name}'")
        return env[e.name]
    if isinstance(e, Neg):
        return -evaluate(e.arg, env)
    if isinstance(e, Bin):
        a, b = evaluate(e.left, env), evaluate(e.right, env)
        if e.op == "+":
            return a + b
        if e.op == "-":
            return a - b
        if e.op == "*":
            return a * b
        if e.op == "//":
            return _fdiv(a, b)
        if e.op == "%":
            return a % b
        return a / b
    if isinstance(e, Call):
        vals = [evaluate(a, env) for a in e.args]
        if e.fn == "min":
            return min(vals)
        if e.fn == "max":
            return max(vals)
        raise ExprError("size() is not evaluable host-side")
    if isinstance(e, Cmp):
        a, b = evaluate(e.left, env), evaluate(e.right, env)
        return int({"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b, "==": a == b,
                    "!=": a != b}[e.op])
    if isinstance(e, BoolOp):
        vals = [evaluate(a, env) for a in e.args]
        return int(all(vals)) if e.op == "and" else int(any(vals))
    if isinstance(e, Not):
        return int(not evaluate(e.arg, env))
    raise ExprError(f"cannot evaluate {e!r}")


def free_symbols(e: Expr) -> set[str]:
    if isinstance(e, Sym):
        return {e.name}
    if isinstance(e, (Bin, Cmp)):
        return free_symbols(e.left) | free_symbols(e.right)
    if isinstance(e, (Neg, Not)):
        return free_symbols(e.arg)
    if isinstance(e, (Call, BoolOp)):
        out: set[str] = set()
        for a in e.args:
            out |= free_symbols(a)
        return out
    return set()


def substitute(e: Expr, mapping: Mapping[str, Expr]) -> Expr:
    if isinstance(e, Sym):
        return mapping.get(e.name, e)
    if isinstance(e, Bin):
        return Bin(e.op, substitute(e.left, mapping), substitute(e.right, mapping))
    if isinstance(e, Cmp):
        return Cmp(e.op, substitute(e.left, mapping), substitute(e.right, mapping))
    if isinstance(e, Neg):
        return Neg(substitute(e.arg, mapping))
    if isinstance(e, Not):
        return Not(substitute(e.arg, mapping))
    if isinstance(e, Call):
        return Call(e.fn, tuple(substitute(a, mapping) for a in e.args))
    if isinstance(e, BoolOp):
        return BoolOp(e.op, tuple(substitute(a, mapping) for a in e.args))
    return e


# ------------------------------------------------------------------- affine

class Affine:
    """``const + sum(coeff * sym)`` with integer coefficients."""

    __slots__ = ("terms", "const")

    def __init__(self, terms=None, const=0):
        self.terms = {k: v for k, v in (terms or {}).items() if v != 0}
        self.const = const

    def __add__(self, o):
        t = dict(self.terms)
        for k, v in o.terms.items():
            t[k] = t.get(k, 0) + v
        return Affine(t, self.const + o.const)

    def scale(self, c):
        return Affine({k: v * c for k, v in self.terms.items()}, self.const * c)

    def __sub__(self, o):
        return self + o.scale(-1)

    def __eq__(self, o):
        return isinstance(o, Affine) and self.terms == o.terms and self.const == o.const

    def __hash__(self):
        return hash((tuple(sorted(self.terms.items())), self.const))

    def is_const(self):
        return not self.terms

    def only(self, sym):
        """coefficient-1 ``sym + const`` -> const, else None."""
        if set(self.terms) == {sym} and self.terms[sym] == 1:
            return self.const
        return None

    def __repr__(self):
        parts = [f"{v}*{k}" for k, v in sorted(self.terms.items())]
        return " + ".join(parts + [str(self.const)])


def affine(e: Expr) -> Optional[Affine]:
    """Affine decomposition over integer coefficients, or None."""
    if isinstance(e, Num):
        return Affine({}, e.value) if isinstance(e.value, int) else None
    if isinstance(e, Sym):
        return Affine({e.name: 1}, 0)
    if isinstance(e, Neg):
        a = affine(e.arg)
        return a.scale(-1) if a is not None else None
    if isinstance(e, Bin):
        a, b = affine(e.left), affine(e.right)
        if a is None or b is None:
            return None
        if e.op == "+":
            return a + b
        if e.op == "-":
            return a - b
        if e.op == "*":
            if a.is_const():
                return b.scale(a.const)
            if b.is_const():
                return a.scale(b.const)
    return None


def same_value(a: Expr, b: Expr) -> bool:
    """Structural or affine equality."""
    if a == b:
        return True
    fa, fb = affine(a), affine(b)
    return fa is not None and fb is not None and fa == fb
