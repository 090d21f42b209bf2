"""Operand construction by powering: the expression
language of the reference (io.py:1-231) with an injected multiplier.  CPU
tests use the oracle multiplier; tests/test_gpu_parity.py runs the same corpus
with the GPU product."""

from __future__ import annotations

import pytest

from conftest import golden
from oracle import oracle as O
from paper_1303_7425_b200 import default_layout, format_poly, io
from paper_1303_7425_b200.expr import ExprSyntaxError, parse, poly_from_expr, power, variables_of

EXPRS = [e for e in golden()["exprs"] if "^30" not in e["text"]]


def oracle_mul(a, b):
    return O.mul(a, b)


@pytest.mark.parametrize("e", EXPRS, ids=[f"{e['text']}/{e['ctype']}" for e in EXPRS])
def test_expression_corpus_matches_reference(e):
    lay = default_layout(tuple(e["vars"]))
    ct = float if e["ctype"] == "float" else int
    p = poly_from_expr(e["text"], lay, ct, mul=oracle_mul)
    assert p.n == e["n"]
    assert io.poly_digest(p) == e["sha256"]


def test_syntax_errors_and_positions():
    for bad, pos in (("x+", 2), ("(x", 2), ("x^y", 2), ("2x$", 2), ("x)", 1)):
        with pytest.raises(ExprSyntaxError) as err:
            parse(bad)
        assert err.value.pos == pos, bad
    lay = default_layout(("x",))
    with pytest.raises(ExprSyntaxError):
        parse("y", lay.vars)


def test_binary_exponentiation_call_count_and_order():
    calls = []

    def rec(a, b):
        calls.append((a.n, b.n))
        return O.mul(a, b)

    lay = default_layout(("x",))
    poly_from_expr("(1+x)^5", lay, mul=rec)
    # 5 = 101b: result*base, base^2, base^4, result*base
    assert calls == [(1, 2), (2, 2), (3, 3), (2, 5)]
    assert power(None, 0, None, "one") == "one"


def test_variables_in_order_of_first_appearance():
    assert variables_of("(1+x+y+2*z^2+3*t^3+5*u^5)^2", "(1+u+t)^2") == ("x", "y", "z", "t", "u")
