"""Benchmark-operand construction on the GPU: the expression language of the
reference (io.py:1-231) evaluated with the GPU `mul` injected.

This is SURVEY §8(f) row 1, the caller one step upstream of the hot path.
Every benchmark operand, such as "(1+x+y+2*z^2+3*t^3+5*u^5)^25", is built by
binary exponentiation with a pluggable multiplier (io.py:194-226).

Grammar (the reference's, io.py:12-18):
    expr   := ['-'] term (('+'|'-') term)*      leading '-' means 0 - term
    term   := factor ('*' factor)*
    factor := atom ('^' uint)?
    atom   := uint | name | '(' expr ')'

The AST is plain tuples: ('num', v), ('var', name), ('add'|'sub'|'mul', l, r)
and ('pow', base, n).  Evaluation order matches the reference call for call:
left before right, and `result = mul(result, base)` / `base = mul(base, base)`
in the reference's loop.  So an order-exact multiplier (MulConfig.float_ordered)
reproduces the reference's float operands bit for bit.
"""

from __future__ import annotations

import re

from .core import Polynomial, VarTable, default_layout


class ExprSyntaxError(ValueError):
    def __init__(self, message: str, pos: int):
        super().__init__(f"{message} (at position {pos})")
        self.pos = pos


_TOK = re.compile(r"\s*(?:(?P<int>\d+)|(?P<name>[A-Za-z_]\w*)|(?P<op>[-+*^()]))")


def tokens(text: str) -> list:
    out, pos = [], 0
    while True:
        m = _TOK.match(text, pos)
        if m is None:
            rest = text[pos:].lstrip()
            if rest:
                raise ExprSyntaxError(f"unexpected character {rest[0]!r}", len(text) - len(rest))
            out.append(("end", None, len(text)))
            return out
        kind = m.lastgroup
        val = int(m.group(kind)) if kind == "int" else m.group(kind)
        out.append((val if kind == "op" else kind, val, m.start(kind)))
        pos = m.end()


def parse(text: str, vars: VarTable | None = None):
    toks = tokens(text)
    at = [0]

    def peek():
        return toks[at[0]]

    def take():
        at[0] += 1
        return toks[at[0] - 1]

    def expr():
        if peek()[0] == "-":
            take()
            node = ("sub", ("num", 0), term())
        else:
            node = term()
        while peek()[0] in ("+", "-"):
            op = take()[0]
            node = ("add" if op == "+" else "sub", node, term())
        return node

    def term():
        node = factor()
        while peek()[0] == "*":
            take()
            node = ("mul", node, factor())
        return node

    def factor():
        node = atom()
        if peek()[0] == "^":
            take()
            kind, val, pos = take()
            if kind != "int":
                raise ExprSyntaxError("power must be a literal non-negative integer", pos)
            node = ("pow", node, val)
        return node

    def atom():
        kind, val, pos = take()
        if kind == "int":
            return ("num", val)
        if kind == "name":
            if vars is not None and val not in vars.names:
                raise ExprSyntaxError(f"unknown variable {val!r}", pos)
            return ("var", val)
        if kind == "(":
            node = expr()
            if take()[0] != ")":
                raise ExprSyntaxError("expected ')'", toks[at[0] - 1][2])
            return node
        raise ExprSyntaxError("expected a number, variable or '('", pos)

    node = expr()
    if peek()[0] != "end":
        raise ExprSyntaxError(f"unexpected trailing input {peek()[1]!r}", peek()[2])
    return node


def power(base, n: int, mul, one):
    """Binary exponentiation in the reference's call order (io.py:215-225)."""
    result = one
    while n:
        if n & 1:
            result = mul(result, base)
        n >>= 1
        if n:
            base = mul(base, base)
    return result


def evaluate(node, layout, ctype=int, mul=None):
    """Value of an expression tree.  With the default (GPU) multiplier the
    intermediate products of powering stay array-backed (ArrayPolynomial via
    mul_arrays): no Python int is built until the final result."""
    if mul is None:
        from .arrays import ArrayPolynomial
        from .parmul import MulConfig, mul_arrays
        # float operands are built in the reference's summation order (its
        # default multiplier folds rows in increasing i), so they are the
        # reference's operands bit for bit, not just within tolerance
        cfg = MulConfig(float_ordered=ctype is float)
        out = _evaluate(node, layout, ctype, lambda x, y: mul_arrays(x, y, cfg))
        return out.to_poly() if isinstance(out, ArrayPolynomial) else out
    return _evaluate(node, layout, ctype, mul)


def _lists(p):
    return p.to_poly() if hasattr(p, "to_poly") else p


def _evaluate(node, layout, ctype, mul):
    kind = node[0]
    if kind == "num":
        return Polynomial.constant(layout, node[1], ctype)
    if kind == "var":
        return Polynomial.variable(layout, node[1], ctype)
    if kind == "pow":
        base = _evaluate(node[1], layout, ctype, mul)
        return power(base, node[2], mul, Polynomial.constant(layout, 1, ctype))
    left = _evaluate(node[1], layout, ctype, mul)
    right = _evaluate(node[2], layout, ctype, mul)
    if kind == "add":
        return _lists(left) + _lists(right)
    if kind == "sub":
        return _lists(left) - _lists(right)
    return mul(left, right)


def poly_from_expr(text: str, layout, ctype=int, mul=None):
    """reference io.poly_from_expr with the GPU product as the default `mul`."""
    return evaluate(parse(text, layout.vars), layout, ctype, mul)


def variables_of(*texts) -> tuple:
    """Variable names in order of first appearance (reference io.expr_var_names)."""
    seen = []
    for t in texts:
        for kind, val, _ in tokens(t):
            if kind == "name" and val not in seen:
                seen.append(val)
    return tuple(seen)


# the reference's benchmark examples (service/app.py:38-42)
BENCH_EXAMPLES = {
    1: ("(1+x+y+z+t)^{p}", "(1+x+y+z+t)^{p}+1"),
    2: ("(1+x+y+2*z^2+3*t^3+5*u^5)^{p}", "(1+u+t+2*z^2+3*y^3+5*x^5)^{p}"),
    3: ("(1+u^2+v+w^2+x-y^2)^{p}", "(1+u+v^2+w+x^2+y^3)^{p}+1"),
}


def bench_pair(example: int, p: int, ctype=int, mul=None):
    """The reference's /bench operands (service/app.py:38-42, 46-85: vars in
    order of first appearance across both expressions)."""
    fa, fb = (t.format(p=p) for t in BENCH_EXAMPLES[example])
    lay = default_layout(variables_of(fa, fb))
    return poly_from_expr(fa, lay, ctype, mul), poly_from_expr(fb, lay, ctype, mul)
