"""Generate golden vectors by running the REFERENCE implementation.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/cases.json: operands and the reference's own product
(`polymul.parmul.mul`, default MulConfig unless noted) for a corpus that
follows the reference's tests -- rand_poly with duplicate/zero input terms
(conftest.py:24-36), random_sparse (parmul.py:129-156) as in acceptance
criterion 3 (test_acceptance.py:129-161), lex order, 14 variables with 4-bit
fields, narrow custom layouts, floats with inf/nan, cancellation, explicit
split sets including ones whose first bound is above the minimum sum
(SURVEY.md 8a item 6), plus select_grid bounds and count_ops values.

The reference is imported only here; the committed JSON travels, the
reference does not.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import random
import sys
from pathlib import Path

from polymul.core import Layout, Polynomial, SENTINEL, VarTable, default_layout
from polymul.parmul import MulConfig, mul, random_sparse
from polymul.split import GridParams, SplitSet, count_ops, find_edge, select_grid

OUT = Path(__file__).resolve().parent / "cases.json.gz"


def enc_coef(c):
    if isinstance(c, float):
        if math.isnan(c):
            return "nan"
        if math.isinf(c):
            return "inf" if c > 0 else "-inf"
        return repr(c)
    return str(c)


def enc_poly(p):
    lay = p.layout
    return {"exps": [str(e) for e in p.exps], "coeffs": [enc_coef(c) for c in p.coeffs]}


def product_digest(exps, coeffs) -> str:
    """sha256 over "<packed exp> <coeff>\n" lines (SURVEY.md Appendix A format;
    floats rendered with repr, specials as nan/inf/-inf)."""
    h = hashlib.sha256()
    for e, c in zip(exps, coeffs):
        h.update(f"{e} {enc_coef(c)}\n".encode())
    return h.hexdigest()


def enc_product(p):
    out = {"n": p.n, "sha256": product_digest(p.exps, p.coeffs)}
    if p.n <= 200:
        out.update(enc_poly(p))
    return out


def enc_layout(lay):
    return {"vars": list(lay.vars.names), "order": lay.order, "var_bits": list(lay.var_bits),
            "deg_bits": lay.deg_bits}


def rand_poly(rng, m, terms, max_deg=8, ctype=int, layout=None):
    if layout is None:
        layout = default_layout([f"x{i}" for i in range(1, m + 1)])
    pairs = []
    for _ in range(terms):
        c = rng.randint(-50, 50) or 7
        pairs.append((ctype(c), tuple(rng.randint(0, max_deg) for _ in range(m))))
    return Polynomial(layout, pairs, ctype)


def safe_max_deg(m, terms, dense):
    d = 1
    while (d + 1) ** m < 2 * terms:
        d += 1
    if not dense:
        d *= 3
    cap = {1: 4000, 2: 2000, 3: 500, 4: 500, 5: 120, 6: 40, 7: 25, 8: 15}[m]
    return min(d, cap)


def main():
    rng = random.Random(20260811)
    cases = []

    def add(name, a, b, cfg=None, split=None):
        prod = mul(a, b, cfg or MulConfig(), split=split)
        cases.append({"name": name, "layout": enc_layout(a.layout),
                      "ctype": "float" if a.ctype is float else "int",
                      "a": enc_poly(a), "b": enc_poly(b),
                      "split": None if split is None else [str(x) for x in split.bounds],
                      "product": enc_product(prod)})

    # rand_poly corpus (duplicates/zeros canonicalized on input)
    for k in range(40):
        m = rng.randint(1, 6)
        a = rand_poly(rng, m, rng.randint(1, 60), 6)
        b = rand_poly(rng, m, rng.randint(1, 60), 6)
        add(f"rand_{k}", a, b, MulConfig(l=rng.choice([1, 2, 7, 64])))
    # acceptance-criterion-3 style (random_sparse, dense and sparse exponents)
    arng = random.Random(0xACCE97)
    for idx in range(60):
        m = (idx % 8) + 1
        terms = arng.randint(1, 120) if idx % 5 else arng.randint(120, 400)
        tb = arng.randint(1, terms)
        if terms * tb > 8_000:
            tb = max(1, 8_000 // terms)
        dense = idx % 2 == 0
        a = random_sparse(arng.randrange(1 << 30), m, terms, safe_max_deg(m, terms, dense))
        b = random_sparse(arng.randrange(1 << 30), m, tb, safe_max_deg(m, tb, dense))
        add(f"sparse_{idx}", a, b)
    # floats, including specials
    for k in range(10):
        m = rng.randint(1, 4)
        a = rand_poly(rng, m, rng.randint(5, 50), 6, float)
        b = rand_poly(rng, m, rng.randint(5, 50), 6, float)
        add(f"float_{k}", a, b)
    lay = default_layout(("x",))
    x = Polynomial.variable(lay, "x", float)
    add("float_inf", Polynomial.constant(lay, float("inf"), float) + x,
        Polynomial.constant(lay, 1.0, float) - x)
    add("float_nan", Polynomial.constant(lay, float("nan"), float) + x, x + x)
    add("float_tiny_cancel", Polynomial(lay, [(1e16, (1,)), (1.0, (0,))], float),
        Polynomial(lay, [(1.0, (1,)), (-1e16, (0,))], float))
    # cancellation / zero results
    lay2 = default_layout(("x", "y"))
    X = Polynomial.variable(lay2, "x")
    Y = Polynomial.variable(lay2, "y")
    add("cancel_diff_squares", X - Y, X + Y)
    add("cancel_all", Polynomial(lay2, [(1, (1, 0)), (1, (0, 1))]),
        Polynomial(lay2, [(1, (1, 0)), (-1, (0, 1))]))
    add("monomials", X, Y)
    # big ints
    big = Polynomial(lay2, [(3 ** 60, (1, 0)), (-(2 ** 90), (0, 1)), (7, (0, 0))])
    add("bigint_90", big, big)
    add("bigint_mixed", big, X + Y)
    # lex order, 14 variables, narrow layouts
    llex = default_layout(("x", "y", "z"), order="lex")
    add("lex_3", rand_poly(rng, 3, 40, 8, layout=llex), rand_poly(rng, 3, 35, 8, layout=llex))
    l14 = default_layout([f"v{i}" for i in range(14)])
    add("vars_14", rand_poly(rng, 14, 25, 3, layout=l14), rand_poly(rng, 14, 25, 3, layout=l14))
    narrow = Layout.for_max_degrees(VarTable(("x", "y")), (30, 30))
    add("narrow_layout", rand_poly(rng, 2, 30, 15, layout=narrow),
        rand_poly(rng, 2, 30, 15, layout=narrow))
    nlex = Layout.for_max_degrees(VarTable(("x", "y", "z")), (20, 9, 9), order="lex")
    add("narrow_lex", rand_poly(rng, 3, 30, 4, layout=nlex), rand_poly(rng, 3, 30, 4, layout=nlex))
    m1 = default_layout(("x",))
    add("univariate_wide", random_sparse(5, 1, 120, 4000, layout=m1),
        random_sparse(6, 1, 90, 4000, layout=m1))
    # explicit splits (test_parmul.py:90-102 and the lower-bound semantics)
    a = rand_poly(rng, 3, 30, 6)
    b = rand_poly(rng, 3, 30, 6)
    realized = sorted({ea + eb for ea in a.exps for eb in b.exps})
    for k in range(4):
        picks = rng.sample(realized, rng.randint(0, min(12, len(realized))))
        add(f"split_cover_{k}", a, b, split=SplitSet(sorted(set(picks) | {realized[0], SENTINEL})))
    add("split_loose", a, b, split=SplitSet(sorted({realized[0], realized[-1] + 1, SENTINEL - 5,
                                                      SENTINEL})))
    add("split_above_min", a, b, split=SplitSet([realized[len(realized) // 2], SENTINEL]))
    add("split_between", a, b, split=SplitSet([realized[len(realized) // 3] + 1, SENTINEL]))
    one_x = Polynomial.constant(lay, 1) + Polynomial.variable(lay, "x")
    add("split_survey_example", one_x, one_x,
        split=SplitSet([lay.pack((1,)), SENTINEL]))  # (1+x)^2 -> 2x + x^2

    # select_grid / count_ops goldens
    grids = []
    for k in range(8):
        m = rng.randint(1, 5)
        a = rand_poly(rng, m, rng.randint(5, 200), 7)
        b = rand_poly(rng, m, rng.randint(5, 200), 7)
        l = rng.choice([1, 3, 8, 64])
        bounds = select_grid(a, b, GridParams(l)).bounds
        ops = [sum(j1 - j0 + 1 for j0, j1 in zip(e.lmin, e.lmax) if j0 <= j1)
               for e in (find_edge(a, b, bounds[q], bounds[q + 1]) for q in range(len(bounds) - 1))]
        assert sum(ops) == a.n * b.n
        grids.append({"layout": enc_layout(a.layout), "a": enc_poly(a), "b": enc_poly(b), "l": l,
                      "bounds": [str(x) for x in bounds], "ops": ops})
    # expression corpus (reference test_io.py:108-140 plus benchmark shapes):
    # sha256 of the reference's format_poly(poly_from_expr(text)) with its own mul
    from polymul.io import format_poly, poly_from_expr
    fast = lambda a, b: mul(a, b, MulConfig(l=16, c=8))
    exprs = []
    corpus = [("0", "x y z"), ("7", "x y z"), ("x", "x y z"), ("x+y", "x y z"), ("x-x", "x y z"),
              ("-x", "x y z"), ("2*x", "x y z"), ("x*y*z", "x y z"), ("x^3", "x y z"),
              ("(x+y)^2", "x y z"), ("(1+x)*(1-x)", "x y z"), ("1+x*y^3", "x y z"),
              ("(x+y)*(y+z)", "x y z"), ("((x))", "x y z"), ("x^2*x^3", "x y z"),
              ("(1+x+y+z)^3-(1+x+y+z)^3", "x y z"), ("3-2", "x y z"), ("2^3", "x y z"),
              ("1-x^2", "x y z"), ("(2*x+3*y)^2", "x y z"),
              ("(1+x+y+z+t)^8", "x y z t"), ("(1+x+y+z+t)^8+1", "x y z t"),
              ("(1+x+y+2*z^2+3*t^3+5*u^5)^5", "x y z t u"),
              ("(1+u^2+v+w^2+x-y^2)^5", "u v w x y"), ("(1+u+v^2+w+x^2+y^3)^5+1", "u v w x y")]
    for text, names in corpus:
        for ct in (int, float):
            lay = default_layout(tuple(names.split()))
            p_ = poly_from_expr(text, lay, ct, mul=fast)
            exprs.append({"text": text, "vars": names.split(), "ctype": ct.__name__, "n": p_.n,
                          "sha256": hashlib.sha256(format_poly(p_).encode()).hexdigest()})
    # the Fateman n=30 float operands exactly as the reference builds them
    # (repeated squaring in float); their digest pins GPU float_ordered powering
    lay4 = default_layout(("x", "y", "z", "t"))
    for text in ("(1+x+y+z+t)^30", "(1+x+y+z+t)^30+1"):
        p_ = poly_from_expr(text, lay4, float, mul=fast)
        exprs.append({"text": text, "vars": ["x", "y", "z", "t"], "ctype": "float", "n": p_.n,
                      "sha256": hashlib.sha256(format_poly(p_).encode()).hexdigest()})
    OUT.write_bytes(gzip.compress(json.dumps({"generator": "tests/golden/make_golden.py",
                               "reference": "polymul 0.1.0 (/root/reference/pkg)",
                               "cases": cases, "grids": grids, "exprs": exprs},
                               separators=(",", ":")).encode(), 9))
    print(f"wrote {len(cases)} product cases and {len(grids)} grid cases to {OUT}", file=sys.stderr)


if __name__ == "__main__":
    main()
