"""Host-side logic of the drop-in: the polynomial data model (reference
core.py semantics), configuration validation, marshaling, grid sampling and
the cluster partition -- all without a GPU."""

from __future__ import annotations

import random

import numpy as np
import pytest

from conftest import golden, dec_layout, dec_poly
from oracle import oracle as O
from paper_1303_7425_b200 import (SENTINEL, ExponentOverflowError, GridParams, Layout, MulConfig,
                                  Polynomial, SplitSet, VarTable, check_product_fits,
                                  default_layout, format_poly, partition_by_ops, select_grid)
from paper_1303_7425_b200 import _native as N
from paper_1303_7425_b200.cluster import block, rank_range
from paper_1303_7425_b200.parmul import Operand, int_coeff_array, limbs_to_ints


def ref_key(order, vec):
    return (sum(vec), vec) if order == "grlex" else vec


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8, 14])
@pytest.mark.parametrize("order", ["grlex", "lex"])
def test_pack_roundtrip_and_order(m, order, rng):
    lay = default_layout([f"v{i}" for i in range(m)], order)
    vecs = [tuple(rng.randint(0, 3) for _ in range(m)) for _ in range(60)]
    for v in vecs:
        assert lay.unpack(lay.pack(v)) == v
    packed = sorted(vecs, key=lambda v: lay.pack(v))
    assert packed == sorted(vecs, key=lambda v: ref_key(order, v))


def test_layout_defaults_match_reference_widths():
    assert default_layout(("x", "y", "z", "t")).fields() == [(48, 16), (36, 12), (24, 12), (12, 12), (0, 12)]
    assert default_layout(("x", "y", "z", "t", "u")).fields() == [(50, 14), (40, 10), (30, 10), (20, 10), (10, 10), (0, 10)]
    lex = default_layout(("x", "y"), "lex")
    assert lex.fields() == [(32, 32), (0, 32)] and lex.max_vector() == ((1 << 32) - 2, (1 << 32) - 1)
    assert Layout.for_max_degrees(VarTable(("x", "y")), (30, 30)).var_bits == (5, 5)


def test_overflow_detected_not_wrapped():
    lay = default_layout(("x",))
    with pytest.raises(ExponentOverflowError):
        lay.pack((lay.max_vector()[0] + 1,))
    a = Polynomial(lay, [(1, (lay.max_vector()[0] // 2 + 1,))])
    with pytest.raises(ExponentOverflowError):
        check_product_fits(a, a)


def test_canonicalize_drops_zeros_and_merges(rng):
    lay = default_layout(("x", "y"))
    p = Polynomial(lay, [(2, (1, 0)), (-2, (1, 0)), (3, (0, 1)), (4, (0, 1)), (0, (2, 2))])
    assert p.coeffs == [7] and p.exps == [lay.pack((0, 1))]
    p.validate()


def test_config_validation():
    assert MulConfig() == MulConfig(l=64, c=1, merger="heap")
    for kw in (dict(l=0), dict(c=0), dict(merger="quick"), dict(path="fast")):
        with pytest.raises(ValueError):
            MulConfig(**kw)
    with pytest.raises(ValueError):
        SplitSet([1, 2])
    with pytest.raises(ValueError):
        SplitSet([3, 2, SENTINEL])
    with pytest.raises(ValueError):
        GridParams(0)


def test_select_grid_matches_reference_goldens():
    for g in golden()["grids"]:
        lay = dec_layout(g["layout"])
        a = dec_poly(g["a"], lay, int)
        b = dec_poly(g["b"], lay, int)
        assert select_grid(a, b, GridParams(g["l"])).bounds == [int(x) for x in g["bounds"]]


def test_partition_by_ops_greedy_bound():
    rng = random.Random(7)
    for _ in range(300):
        n = rng.randint(1, 60)
        ops = [rng.randint(0, 1000) for _ in range(n)]
        nodes = rng.randint(1, 9)
        plan = partition_by_ops(ops, nodes)
        assert plan.ranges[0][0] == 0 and plan.ranges[-1][1] == n
        assert all(plan.ranges[r][1] == plan.ranges[r + 1][0] for r in range(nodes - 1))
        total = sum(ops)
        assert max(plan.loads()) <= total / nodes + max(ops) + 1e-9
        assert sum(plan.loads()) == total


def test_block_slices_tile_the_intervals():
    for n in range(0, 50):
        for nodes in range(1, 9):
            cover = []
            for r in range(nodes):
                lo, hi = block(n, nodes, r)
                cover.extend(range(lo, hi))
            assert cover == list(range(n))


def test_rank_ranges_cover_the_exponent_space():
    bounds = [5, 9, 20, 33, SENTINEL]
    plan = partition_by_ops([4, 4, 4, 4], 3)
    rr = [rank_range(bounds, plan, r) for r in range(3)]
    assert rr[0][0] == 0 and rr[-1][1] == SENTINEL
    for (l0, h0), (l1, h1) in zip(rr, rr[1:]):
        assert h0 == l1


def test_int_marshaling_roundtrip():
    vals = [0, 1, -1, (1 << 63) - 1, -(1 << 63)]
    arr, kind = int_coeff_array(vals)
    assert kind == N.I64 and arr.tolist() == vals
    big = [(1 << 100) + 5, -(1 << 126), 3, -7]
    arr, kind = int_coeff_array(big)
    assert kind == N.I128
    assert limbs_to_ints(arr, 2) == big
    three = np.array([[5, 0, 0], [(1 << 64) - 1, (1 << 64) - 1, (1 << 64) - 1],
                      [0, 1, 0], [0, 0, (1 << 64) - 1]], dtype=np.uint64)
    assert limbs_to_ints(three, 3) == [5, -1, 1 << 64, -(1 << 128)]


def test_operand_marshaling_of_reference_style_objects():
    lay = default_layout(("x", "y"))
    p = Polynomial(lay, [(1.5, (1, 0)), (-2.0, (0, 3))], float)
    op = Operand.from_poly(p)
    assert op.kind == N.F64 and op.exps.tolist() == p.exps and op.coef.tolist() == p.coeffs


def test_format_poly_matches_reference_text():
    lay = default_layout(("x", "y"))
    p = Polynomial(lay, [(3, (1, 0)), (-2, (0, 2))])
    assert format_poly(p) == "vars x y\n3 1 0\n-2 0 2\n"
    q = Polynomial(lay, [(2.0, (0, 0))], float)
    assert format_poly(q) == "vars x y\n2.0 0 0\n"


def test_oracle_count_ops_sums_to_all_pairs(rng):
    lay = default_layout(("x", "y", "z"))
    a = Polynomial(lay, [(1, (rng.randint(0, 5), rng.randint(0, 5), rng.randint(0, 5))) for _ in range(40)])
    b = Polynomial(lay, [(1, (rng.randint(0, 5), rng.randint(0, 5), rng.randint(0, 5))) for _ in range(30)])
    bounds = select_grid(a, b, GridParams(5)).bounds
    ops = [O.count_ops(a, b, bounds[k], bounds[k + 1]) for k in range(len(bounds) - 1)]
    assert sum(ops) == a.n * b.n


def test_limb_marshaling_helper_matches_python_ints():
    """csrc/pylimbs.c (C marshaling of result limbs) == the pure-Python conversion."""
    import random
    from paper_1303_7425_b200 import parmul
    from paper_1303_7425_b200.arrays import int_limbs
    from paper_1303_7425_b200.build import build_pylimbs
    build_pylimbs()
    parmul._PYLIMBS = None
    assert parmul._pylimbs() is not None
    R = random.Random(3)
    for nl in (1, 2, 3):
        B = 64 * nl
        vals = [R.randrange(-2 ** (B - 1), 2 ** (B - 1)) >> R.randrange(0, B) for _ in range(20000)]
        vals += [0, -1, 2 ** (B - 1) - 1, -2 ** (B - 1), 2 ** 63 - 1, -2 ** 63]
        vals = [v for v in vals if -2 ** (B - 1) <= v < 2 ** (B - 1)]
        arr, _ = int_limbs(vals, nl)
        assert parmul.limbs_to_ints(arr, nl) == vals


def test_polyfile_reader_mirrors_reference_rules():
    """parse_poly (reference io.py:251-290): round trip of format_poly, ctype
    inference, duplicate lines combined, and the reference's error messages."""
    from paper_1303_7425_b200 import PolyIOError, format_poly, parse_poly
    from conftest import golden_cases
    for _, a, b, _, _ in golden_cases()[::9]:
        for p in (a, b):
            q = parse_poly(format_poly(p), p.layout)
            assert q.exps == p.exps and q.ctype is p.ctype
            assert [repr(c) for c in q.coeffs] == [repr(c) for c in p.coeffs]
    p = parse_poly("# c\nvars x y\n2 1 0\n3 1 0\n-5 0 0\n")
    assert p.ctype is int and p.n == 2 and p.coeffs == [-5, 5]
    assert parse_poly("vars x\n1.5 2\n").ctype is float
    for text, msg in [("1 2\n", "line 1: expected 'vars <name>...' header"),
                      ("", "missing 'vars' header line"),
                      ("vars x\n1 2 3\n", "line 2: expected coefficient plus 1 exponents, got 3 fields"),
                      ("vars x\n1 -2\n", "line 2: negative exponent"),
                      ("vars x\nq 2\n", "line 2: malformed number")]:
        with pytest.raises(PolyIOError) as exc:
            parse_poly(text)
        assert str(exc.value) == msg
