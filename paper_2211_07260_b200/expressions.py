"""Restriction / user-metric expression language.

Semantics follow the reference interpreter (``pkg/src/jouletune/expressions.py:
22-160``): Python syntax limited to numeric/bool literals, names, the seven
arithmetic operators (``/`` is true division), unary ``- + not``, ``and``/``or``
returning operand values, chained comparisons and the ``min``/``max``/``abs``
builtins. Unknown names raise :class:`UnknownNameError` at evaluation time.

Implementation differs: instead of walking the AST on every call, the
validated tree is lowered once into a tree of Python closures. Search-space
enumeration evaluates restrictions hundreds of thousands of times (a CLBlast
SGEMM space is ~10^5-10^6 raw combinations), so the one-off lowering pays.
"""

from __future__ import annotations

import ast
import operator
from typing import Callable, Mapping

from .errors import ExpressionError, UnknownNameError

__all__ = ["Expression"]

_ARITH = {
    ast.Add: operator.add,
    ast.Sub: operator.sub,
    ast.Mult: operator.mul,
    ast.Div: operator.truediv,
    ast.FloorDiv: operator.floordiv,
    ast.Mod: operator.mod,
    ast.Pow: operator.pow,
}
_CMP = {
    ast.Eq: operator.eq,
    ast.NotEq: operator.ne,
    ast.Lt: operator.lt,
    ast.LtE: operator.le,
    ast.Gt: operator.gt,
    ast.GtE: operator.ge,
}
_UNARY = {ast.USub: operator.neg, ast.UAdd: operator.pos, ast.Not: operator.not_}
_BUILTINS = {"abs": abs, "max": max, "min": min}

Env = Mapping[str, object]
Thunk = Callable[[Env], object]


class _Lowering:
    """Validates a parsed tree and turns it into closures in one pass."""

    def __init__(self, source: str):
        self.source = source
        self.names: set[str] = set()

    def fail(self, what: str) -> ExpressionError:
        return ExpressionError(f"{what} in {self.source!r}")

    def lower(self, node: ast.AST) -> Thunk:
        kind = type(node)
        if kind is ast.Constant:
            value = node.value
            if not isinstance(value, (bool, int, float)):
                raise self.fail(f"unsupported syntax {kind.__name__!r}")
            return lambda env, _v=value: _v
        if kind is ast.Name:
            return self._name(node.id)
        if kind is ast.BinOp and type(node.op) in _ARITH:
            fn = _ARITH[type(node.op)]
            lhs, rhs = self.lower(node.left), self.lower(node.right)
            return lambda env: fn(lhs(env), rhs(env))
        if kind is ast.UnaryOp and type(node.op) in _UNARY:
            fn = _UNARY[type(node.op)]
            arg = self.lower(node.operand)
            return lambda env: fn(arg(env))
        if kind is ast.BoolOp:
            parts = [self.lower(v) for v in node.values]
            return _all_of(parts) if isinstance(node.op, ast.And) else _any_of(parts)
        if kind is ast.Compare:
            if not all(type(op) in _CMP for op in node.ops):
                raise self.fail("unsupported comparison")
            first = self.lower(node.left)
            chain = [(_CMP[type(op)], self.lower(c)) for op, c in zip(node.ops, node.comparators)]
            return _comparison(first, chain)
        if kind is ast.Call and isinstance(node.func, ast.Name) and not node.keywords:
            fname = node.func.id
            if fname not in _BUILTINS:
                raise ExpressionError(
                    f"unsupported function {fname!r} in {self.source!r}; "
                    f"allowed: {sorted(_BUILTINS)}"
                )
            fn = _BUILTINS[fname]
            args = [self.lower(a) for a in node.args]
            return lambda env: fn(*[a(env) for a in args])
        raise self.fail(f"unsupported syntax {kind.__name__!r}")

    def _name(self, name: str) -> Thunk:
        self.names.add(name)
        source = self.source

        def lookup(env: Env):
            try:
                return env[name]
            except KeyError:
                raise UnknownNameError(name, f"expression {source!r}") from None

        return lookup


def _all_of(parts):
    def run(env):
        value = True
        for part in parts:
            value = part(env)
            if not value:
                break
        return value

    return run


def _any_of(parts):
    def run(env):
        value = False
        for part in parts:
            value = part(env)
            if value:
                break
        return value

    return run


def _comparison(first, chain):
    def run(env):
        left = first(env)
        for op, getter in chain:
            right = getter(env)
            if not op(left, right):
                return False
            left = right
        return True

    return run


class Expression:
    """A validated, pre-compiled expression over named scalars.

    ``names`` is the set of identifiers it reads, used by search spaces to
    check restrictions against their parameters and to schedule early
    pruning during enumeration.
    """

    __slots__ = ("source", "names", "_fn")

    def __init__(self, source: str):
        if not isinstance(source, str) or not source.strip():
            raise ExpressionError(f"empty or non-string expression: {source!r}")
        try:
            tree = ast.parse(source, mode="eval")
        except SyntaxError as exc:
            raise ExpressionError(f"cannot parse {source!r}: {exc.msg}") from exc
        lowering = _Lowering(source)
        self._fn = lowering.lower(tree.body)
        self.source = source
        self.names = frozenset(lowering.names)

    def evaluate(self, env: Env):
        return self._fn(env)

    __call__ = evaluate

    def __repr__(self):
        return f"Expression({self.source!r})"

    def __eq__(self, other):
        return isinstance(other, Expression) and other.source == self.source

    def __hash__(self):
        return hash(self.source)
