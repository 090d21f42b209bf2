"""Benchmark operands in closed form (no CPU multiplication).

Fateman:         f = (1+x+y+z+t)^p, g = f + 1            (app.py:39 example 1)
Monagan-Pearce:  f = (1+x+y+2z^2+3t^3+5u^5)^p,
                 g = (1+u+t+2z^2+3y^3+5x^5)^p            (app.py:40 example 2)

Each power of a sum of distinct monomials c_k*m_k is expanded by the
multinomial theorem: the terms are the compositions (e_0..e_r) of p, with
coefficient p!/prod(e_k!) * prod(c_k^e_k) and exponent sum_k e_k*m_k.  For
these bases distinct compositions give distinct monomials, so no term
combines.  Integer operands equal the reference's `poly_from_expr(..., int)`
exactly; float operands are the correctly rounded exact values (the
reference's float expansion rounds during repeated squaring, which can differ
in the last bit once coefficients exceed 2^53).
"""

from __future__ import annotations

from math import factorial

import numpy as np

from .core import Polynomial, default_layout

FATEMAN_VARS = ("x", "y", "z", "t")
MP_VARS = ("x", "y", "z", "t", "u")


def _compositions(total: int, parts: int):
    if parts == 1:
        yield (total,)
        return
    for k in range(total, -1, -1):
        for rest in _compositions(total - k, parts - 1):
            yield (k,) + rest


def power_of_sum(layout, base, p: int, ctype=int) -> Polynomial:
    """(sum_k c_k * x^v_k)^p for monomials v_k that are pairwise
    'independent' (distinct compositions -> distinct exponents)."""
    m = layout.vars.m
    fact = [factorial(k) for k in range(p + 1)]
    acc = {}
    for comp in _compositions(p, len(base)):
        coeff = fact[p]
        vec = [0] * m
        for e, (c, v) in zip(comp, base):
            coeff //= fact[e]
        for e, (c, v) in zip(comp, base):
            coeff *= c ** e
            for q in range(m):
                vec[q] += e * v[q]
        key = layout.pack(tuple(vec))
        acc[key] = acc.get(key, 0) + coeff
    exps = sorted(acc)
    coeffs = [acc[e] for e in exps]
    if ctype is float:
        coeffs = [float(c) for c in coeffs]
    return Polynomial._from_sorted(layout, exps, coeffs, ctype)


def _unit(m, q, k=1):
    v = [0] * m
    v[q] = k
    return tuple(v)


def fateman(p: int, ctype=int):
    lay = default_layout(FATEMAN_VARS)
    base = [(1, (0, 0, 0, 0))] + [(1, _unit(4, q)) for q in range(4)]
    f = power_of_sum(lay, base, p, ctype)
    g = f + Polynomial.constant(lay, 1, ctype)
    return f, g


def monagan_pearce(p: int, ctype=int):
    lay = default_layout(MP_VARS)
    x, y, z, t, u = range(5)
    fb = [(1, (0,) * 5), (1, _unit(5, x)), (1, _unit(5, y)), (2, _unit(5, z, 2)),
          (3, _unit(5, t, 3)), (5, _unit(5, u, 5))]
    gb = [(1, (0,) * 5), (1, _unit(5, u)), (1, _unit(5, t)), (2, _unit(5, z, 2)),
          (3, _unit(5, y, 3)), (5, _unit(5, x, 5))]
    return power_of_sum(lay, fb, p, ctype), power_of_sum(lay, gb, p, ctype)


CONFIGS = {
    "fateman10": lambda ct=int: fateman(10, ct),
    "fateman20": lambda ct=int: fateman(20, ct),
    "fateman30": lambda ct=int: fateman(30, ct),
    "mp12": lambda ct=int: monagan_pearce(12, ct),
    "mp25": lambda ct=int: monagan_pearce(25, ct),
}


def reference_float_operands(name: str):
    """The reference's float operands of a config: its poly_from_expr with
    ctype float powers the expression by repeated squaring in float
    (io.py:215-225), so coefficients above 2^53 carry that rounding and differ
    from the correctly rounded closed form.  Built here by the GPU powering
    in the reference's summation order (expr.poly_from_expr), which
    reproduces them bit for bit (tests/test_gpu_parity.py)."""
    from .expr import poly_from_expr
    p = int(name.lstrip("fatemanp"))
    if name.startswith("fateman"):
        lay = default_layout(FATEMAN_VARS)
        base = "(1+x+y+z+t)^%d" % p
        return poly_from_expr(base, lay, float), poly_from_expr(base + "+1", lay, float)
    lay = default_layout(MP_VARS)
    return (poly_from_expr("(1+x+y+2*z^2+3*t^3+5*u^5)^%d" % p, lay, float),
            poly_from_expr("(1+u+t+2*z^2+3*y^3+5*x^5)^%d" % p, lay, float))

