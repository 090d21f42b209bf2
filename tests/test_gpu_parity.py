"""Parity of the CUDA library with the reference (through the C ABI).

Integers: bit-exact (exponents, order, coefficients).  Floats: bit-exact in
float_ordered mode (the reference's summation order); otherwise within the
rigorous reordering bound |c_gpu - c_ref| <= 2*k*2^-53*sum_j |a_i b_j| with k
the number of products of the term.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import digests, golden_cases, product_digest
from paper_1303_7425_b200 import (CoefficientOverflowError, ExponentOverflowError, MulConfig,
                                  Polynomial, benchpolys, default_layout, io, mul)
from paper_1303_7425_b200.parmul import Operand, native_mul
from paper_1303_7425_b200.split import GridParams, SplitSet, select_grid

pytestmark = pytest.mark.gpu
CASES = golden_cases()


def _check(got, want, ordered_float=True, a=None, b=None):
    assert got.n == want["n"], f"{got.n} terms vs {want['n']}"
    if got.ctype is int or ordered_float:
        assert product_digest(got.exps, got.coeffs) == want["sha256"]
    elif "exps" in want:
        assert got.exps == [int(e) for e in want["exps"]]


@pytest.mark.parametrize("path", ["auto", "sort", "bucket", "small"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_golden_cases(case, path):
    name, a, b, split, want = case
    cfg = MulConfig(path=path, float_ordered=True)
    got = mul(a, b, cfg, split=None if split is None else SplitSet(split))
    _check(got, want)


@pytest.mark.parametrize("case", [c for c in CASES if c[1].ctype is int], ids=lambda c: c[0])
def test_golden_cases_dense_when_applicable(case):
    name, a, b, split, want = case
    try:
        got = mul(a, b, MulConfig(path="dense"), split=None if split is None else SplitSet(split))
    except Exception as exc:  # key span too wide for the sumset bitmap: the dense path refuses loudly
        assert "dense path" in str(exc)
        return
    _check(got, want)


@pytest.mark.parametrize("cfg", ["fateman10/int", "fateman20/int", "fateman30/int", "mp12/int",
                                 "fateman10/float"])
@pytest.mark.parametrize("path", ["auto", "sort", "bucket"])
def test_benchmark_digests(cfg, path):
    name, kind = cfg.split("/")
    f, g = benchpolys.CONFIGS[name](float if kind == "float" else int)
    p = mul(f, g, MulConfig(path=path))
    want = digests()["products"][cfg]
    assert p.n == want["n"]
    assert io.poly_digest(p) == want["sha256"]


@pytest.mark.parametrize("cfg", ["fateman20/float", "mp12/float"])
def test_float_ordered_mode_is_bit_exact(cfg):
    name, _ = cfg.split("/")
    f, g = benchpolys.CONFIGS[name](float)
    p = mul(f, g, MulConfig(float_ordered=True))
    want = digests()["products"][cfg]
    assert p.n == want["n"] and io.poly_digest(p) == want["sha256"]


@pytest.mark.parametrize("name", ["fateman20", "fateman30", "mp12"])
def test_float_fast_mode_within_bound(name):
    f, g = benchpolys.CONFIGS[name](float)
    fast = mul(f, g, MulConfig(path="auto", float_ordered=False))
    exact = mul(f, g, MulConfig(float_ordered=True))
    assert fast.exps == exact.exps
    # all-positive operands: sum|a_i b_j| == the coefficient itself.  k is the
    # term's own product count (rtol 2k*2^-53, k <= 17,151 on F30),
    # counted exactly on the GPU as the product of the all-ones supports
    ones_f = Polynomial._from_sorted(f.layout, f.exps, [1] * f.n, int)
    ones_g = Polynomial._from_sorted(g.layout, g.exps, [1] * g.n, int)
    cnt = mul(ones_f, ones_g)
    assert cnt.exps == exact.exps and sum(cnt.coeffs) == f.n * g.n
    k = np.asarray(cnt.coeffs, dtype=np.float64)
    x = np.asarray(fast.coeffs)
    y = np.asarray(exact.coeffs)
    bound = 2 * k * 2.0 ** -53 * np.abs(y)
    assert np.all(np.abs(x - y) <= bound)
    if name == "fateman30":
        assert k.max() == 17151  # SURVEY 8(a) segment-length table


@pytest.mark.parametrize("name,path", [("fateman20", "auto"), ("fateman30", "auto"), ("mp12", "auto"),
                                       ("mp12", "bucket"), ("fateman20", "sort"), ("fateman10", "small")])
def test_float_fast_mode_is_deterministic(name, path):
    """Reference acceptance criterion 8 (test_acceptance.py:237-256):
    repeated float products are bit-identical.  No device path may let a race
    (row claims, atomics) decide a summation order."""
    from paper_1303_7425_b200.parmul import mul_arrays
    f, g = benchpolys.CONFIGS[name](float)
    if path == "small":
        f, g = benchpolys.fateman(2, float)
    runs = [mul_arrays(f, g, MulConfig(path=path, float_ordered=False)) for _ in range(3)]
    e0 = runs[0].exps_array()
    c0 = runs[0].coef_array().view(np.uint64)
    for r in runs[1:]:
        assert np.array_equal(r.exps_array(), e0)
        assert np.array_equal(r.coef_array().view(np.uint64), c0)


@pytest.mark.parametrize("path", ["auto", "bucket", "sort"])
@pytest.mark.parametrize("ordered", [None, False])
def test_mp12_float_sparse_paths_equal_reference_digest(path, ordered):
    """Sparse products fold each term in increasing row on the bucket path
    (owner fold in (key, row) order) and on the sort path (stable radix
    order): the default mode, and the fast mode too, give the reference's
    result bit for bit."""
    from paper_1303_7425_b200.parmul import Operand, native_mul
    f, g = benchpolys.CONFIGS["mp12"](float)
    p = mul(f, g, MulConfig(path=path, float_ordered=ordered))
    want = digests()["products"]["mp12/float"]
    assert p.n == want["n"] and io.poly_digest(p) == want["sha256"]
    if path != "auto":
        raw = native_mul(Operand.from_poly(f), Operand.from_poly(g), f.layout, path=path,
                         float_ordered=bool(ordered))
        assert raw.path == path


def test_default_float_mode_is_the_reference_order():
    """mul() without a config (the drop-in call) reproduces the reference's
    float digests: dense-shaped products skip the dense path."""
    f, g = benchpolys.CONFIGS["fateman20"](float)
    p = mul(f, g)
    want = digests()["products"]["fateman20/float"]
    assert p.n == want["n"] and io.poly_digest(p) == want["sha256"]


def test_default_float_powering_builds_reference_operands():
    """poly_from_expr with the default (GPU) multiplier powers float operands in
    the reference's order (its default naive_mul folds rows in increasing i)."""
    from conftest import golden
    from paper_1303_7425_b200.expr import poly_from_expr
    for e in golden()["exprs"]:
        if e["ctype"] != "float" or "^30" in e["text"]:
            continue
        lay = default_layout(tuple(e["vars"]))
        p = poly_from_expr(e["text"], lay, float)
        assert p.n == e["n"] and io.poly_digest(p) == e["sha256"], e["text"]


def test_mp25_sampled_intervals_match_reference():
    """MP n=25 against the reference's digests of sampled intervals
    (SURVEY.md Appendix A), each interval computed as its own GPU range."""
    import hashlib
    d = digests()["mp25_intervals"]
    f, g = benchpolys.monagan_pearce(25)
    bounds = select_grid(f, g, GridParams(d["grid_l"])).bounds
    assert len(bounds) == d["n_s"]
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    rows = {r["k"]: r for r in d["rows"]}
    ks = list(range(0, 4289, 64)) + [4322]
    combined = hashlib.sha256()
    for k in ks:
        raw = native_mul(A, B, f.layout, lo=bounds[k], hi=bounds[k + 1])
        from paper_1303_7425_b200.parmul import limbs_to_ints
        co = limbs_to_ints(raw.coef, raw.nl)
        h = product_digest(raw.exps.tolist(), co)
        combined.update(h.encode())
        if k in rows:
            assert str(bounds[k]) == rows[k]["lo"] or k == 0
            assert raw.pairs == rows[k]["ops"]
            assert raw.exps.size == rows[k]["terms"]
            assert h == rows[k]["sha256"], f"interval {k}"
    assert combined.hexdigest() == d["combined_sha256"]


def test_errors_and_edge_cases():
    lay = default_layout(("x",))
    x = Polynomial.variable(lay, "x")
    with pytest.raises(ValueError):
        mul(x, Polynomial.variable(default_layout(("y",)), "y"))
    with pytest.raises(ValueError):
        mul(x, Polynomial.variable(lay, "x", float))
    assert mul(x, Polynomial.zero(lay)).is_zero
    assert mul(Polynomial.zero(lay), Polynomial.zero(lay)).is_zero
    half = Polynomial(lay, [(1, (lay.max_total_degree() // 2 + 1,))])
    with pytest.raises(ExponentOverflowError):
        mul(half, half)
    # (1+x)^2 with a split starting at x: the constant term is not formed
    one_x = Polynomial.constant(lay, 1) + x
    p = mul(one_x, one_x, split=SplitSet([lay.pack((1,)), (1 << 64) - 1]))
    assert p.coeffs == [2, 1] and p.exps == [lay.pack((1,)), lay.pack((2,))]


def test_coefficient_width_selection_and_overflow_guard():
    lay = default_layout(("x", "y"))
    a = Polynomial(lay, [((1 << 126) - 1, (1, 0)), (-(1 << 126), (0, 1))])
    # the bound needs 126+126+2 bits > 192 -> refused before launch, never wrapped
    with pytest.raises(CoefficientOverflowError):
        mul(a, a)
    b = Polynomial(lay, [((1 << 80) + 1, (1, 0)), (-(1 << 70), (0, 1))])
    c = Polynomial(lay, [(3, (1, 1)), (-7, (2, 0))])
    want = {}
    for ea, ca in zip(b.exps, b.coeffs):
        for ec, cc in zip(c.exps, c.coeffs):
            want[ea + ec] = want.get(ea + ec, 0) + ca * cc
    got = mul(b, c)
    assert got.exps == sorted(k for k, v in want.items() if v)
    assert got.coeffs == [want[e] for e in got.exps]


def test_result_class_follows_operand_class():
    lay = default_layout(("x", "y"))
    a = Polynomial(lay, [(3, (1, 0)), (5, (0, 1))])
    p = mul(a, a)
    assert type(p) is Polynomial
    p.validate()


def test_mp25_full_product_term_count():
    """Full Monagan-Pearce n=25 product on one GPU (batched sort path):
    312,855,140 terms, left in device memory."""
    import torch
    from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
    d = digests()["mp25_intervals"]
    f, g = benchpolys.monagan_pearce(25)
    dev = torch.device("cuda", 0)
    A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
    r = mul_on_device(A, B, f.layout)
    try:
        assert r.pairs == d["total_ops"]
        assert r.n == d["result_terms"]
    finally:
        r.free()


def test_batched_sort_path_matches_single_batch(monkeypatch):
    """Force tiny batches: the concatenated batches equal the one-shot product."""
    f, g = benchpolys.monagan_pearce(6)
    whole = mul(f, g, MulConfig(path="sort"))
    monkeypatch.setenv("PGPU_BATCH_CAP", "20000")
    batched = mul(f, g, MulConfig(path="sort"))
    assert batched.exps == whole.exps and batched.coeffs == whole.coeffs


@pytest.mark.parametrize("path,name", [("dense", "fateman8"), ("sort", "fateman8"),
                                       ("bucket", "fateman8"), ("bucket", "mp6"), ("sort", "mp6")])
def test_disjoint_ranges_concatenate_to_the_product(path, name):
    """The multi-GPU contract: products restricted to consecutive packed ranges
    [S_k, S_k+1) concatenate to the full product (split.py:5-9)."""
    f, g = benchpolys.fateman(8) if name == "fateman8" else benchpolys.monagan_pearce(6)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    full = native_mul(A, B, f.layout, path=path)
    bounds = select_grid(f, g, GridParams(5)).bounds
    cuts = [0] + bounds[1:-1:3] + [(1 << 64) - 1]
    exps, limbs = [], []
    for lo, hi in zip(cuts, cuts[1:]):
        r = native_mul(A, B, f.layout, lo=lo, hi=hi, path=path)
        exps.append(r.exps)
        limbs.append(r.coef)
    assert np.array_equal(np.concatenate(exps), full.exps)
    assert np.array_equal(np.concatenate(limbs), full.coef)


def test_dense_float_matches_oracle_within_bound(rng):
    from oracle import oracle as O
    from paper_1303_7425_b200.core import Polynomial as P
    lay = default_layout(("x", "y", "z"))
    for _ in range(5):
        a = P(lay, [(rng.uniform(-5, 5), (rng.randint(0, 9), rng.randint(0, 9), rng.randint(0, 9)))
                    for _ in range(300)], float)
        b = P(lay, [(rng.uniform(-5, 5), (rng.randint(0, 9), rng.randint(0, 9), rng.randint(0, 9)))
                    for _ in range(300)], float)
        got = mul(a, b, MulConfig(path="dense", float_ordered=False))
        want = O.mul(a, b)
        absa = P._from_sorted(lay, a.exps, [abs(c) for c in a.coeffs], float)
        absb = P._from_sorted(lay, b.exps, [abs(c) for c in b.coeffs], float)
        mag = dict(zip(*[O.mul(absa, absb).exps, O.mul(absa, absb).coeffs]))
        # terms whose reference sum is exactly 0 are dropped by both; tiny
        # cancellations may survive on one side only, within the bound
        gd = dict(zip(got.exps, got.coeffs))
        wd = dict(zip(want.exps, want.coeffs))
        k = min(a.n, b.n)
        for e in set(gd) | set(wd):
            tol = 2 * k * 2.0 ** -53 * mag[e]
            assert abs(gd.get(e, 0.0) - wd.get(e, 0.0)) <= tol


@pytest.mark.parametrize("path", ["dense", "sort", "bucket"])
def test_int128_operands_signed(path, rng):
    """Operands beyond 63 bits (two-limb int128) with mixed signs."""
    from paper_1303_7425_b200.core import Polynomial as P
    lay = default_layout(("x", "y"))
    big = lambda: rng.choice([-1, 1]) * rng.randint(1 << 70, 1 << 90)
    a = P(lay, [(big(), (rng.randint(0, 20), rng.randint(0, 20))) for _ in range(150)])
    b = P(lay, [(big(), (rng.randint(0, 20), rng.randint(0, 20))) for _ in range(150)])
    want = {}
    for ea, ca in zip(a.exps, a.coeffs):
        for eb, cb in zip(b.exps, b.coeffs):
            want[ea + eb] = want.get(ea + eb, 0) + ca * cb
    got = mul(a, b, MulConfig(path=path))
    assert got.exps == sorted(e for e, v in want.items() if v)
    assert got.coeffs == [want[e] for e in got.exps]


def test_device_resident_api_and_free():
    import torch
    from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
    from paper_1303_7425_b200.parmul import limbs_to_ints
    f, g = benchpolys.fateman(6)
    dev = torch.device("cuda", 0)
    A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
    for _ in range(3):
        r = mul_on_device(A, B, f.layout, stream=torch.cuda.current_stream().cuda_stream, timing=True)
        e, c = r.tensors()
        exps = e.cpu().numpy().view(np.uint64).tolist()
        co = limbs_to_ints(c.cpu().numpy().view(np.uint64), r.nl)
        r.free()
        want = mul(f, g, MulConfig(path="sort"))
        assert exps == want.exps and co == want.coeffs
        assert r.launches > 0 and "numeric" in r.phases


def _gpu_ordered_mul(a, b):
    return mul(a, b, MulConfig(float_ordered=True))


def test_expression_corpus_with_gpu_mul():
    from conftest import golden
    from paper_1303_7425_b200.expr import poly_from_expr
    for e in golden()["exprs"]:
        if "^30" in e["text"]:
            continue
        lay = default_layout(tuple(e["vars"]))
        ct = float if e["ctype"] == "float" else int
        p = poly_from_expr(e["text"], lay, ct, mul=_gpu_ordered_mul)
        assert p.n == e["n"] and io.poly_digest(p) == e["sha256"], e["text"]


def test_fateman30_float_operands_and_product_bit_exact():
    """The reference's float Fateman n=30 operands come from repeated squaring
    in float (io.py:215-225); GPU powering in float_ordered mode reproduces
    them bit for bit, and so the reference's float product digest too."""
    from conftest import golden
    from paper_1303_7425_b200.expr import poly_from_expr
    want = {e["text"]: e for e in golden()["exprs"] if "^30" in e["text"]}
    lay = default_layout(("x", "y", "z", "t"))
    f = poly_from_expr("(1+x+y+z+t)^30", lay, float, mul=_gpu_ordered_mul)
    g = poly_from_expr("(1+x+y+z+t)^30+1", lay, float, mul=_gpu_ordered_mul)
    assert io.poly_digest(f) == want["(1+x+y+z+t)^30"]["sha256"]
    assert io.poly_digest(g) == want["(1+x+y+z+t)^30+1"]["sha256"]
    p = mul(f, g, MulConfig(float_ordered=True))
    d = digests()["products"]["fateman30/float"]
    assert p.n == d["n"] and io.poly_digest(p) == d["sha256"]


@pytest.mark.parametrize("name,want_path", [("mp12", ("bucket",)), ("fateman20", ("bucket", "sort"))])
def test_bucket_path_choice_and_fallback(name, want_path):
    """Sparse MP12 runs on the bucket path.  Fateman 20 forced onto it has
    single keys with up to 3,951 pairs: such bins are reduced in the bucket
    kernel's dense mode, or the batch falls back to the sort path (reported in
    path_used); either way the result is the exact product."""
    f, g = benchpolys.CONFIGS[name](int)
    raw = native_mul(Operand.from_poly(f), Operand.from_poly(g), f.layout, path="bucket")
    assert raw.path in want_path
    ref = native_mul(Operand.from_poly(f), Operand.from_poly(g), f.layout, path="sort")
    assert np.array_equal(raw.exps, ref.exps) and np.array_equal(raw.coef, ref.coef)


def test_bucket_path_float_fast_mode_within_bound():
    f, g = benchpolys.CONFIGS["mp12"](float)
    fast = native_mul(Operand.from_poly(f), Operand.from_poly(g), f.layout, path="bucket")
    exact = native_mul(Operand.from_poly(f), Operand.from_poly(g), f.layout, float_ordered=True)
    assert fast.path == "bucket" and np.array_equal(fast.exps, exact.exps)
    k = 114  # longest MP12 segment
    assert np.all(np.abs(fast.coef - exact.coef) <= 2 * k * 2.0 ** -53 * np.abs(exact.coef))


@pytest.mark.parametrize("ctype", [int, float])
def test_bucket_path_random_sparse_vs_oracle(ctype, rng):
    """Random sparse operands (few repeated keys, signed coefficients) through
    the bucket path against the oracle: exact for ints, within the reordering
    bound for floats."""
    from oracle import oracle as O
    from paper_1303_7425_b200.core import Polynomial as P
    lay = default_layout(("x", "y", "z", "t"))
    for _ in range(3):
        terms = lambda n: [((rng.randint(-10 ** 6, 10 ** 6) if ctype is int else rng.uniform(-3, 3)),
                            tuple(rng.randint(0, 40) for _ in range(4))) for _ in range(n)]
        a, b = P(lay, terms(2000), ctype), P(lay, terms(1500), ctype)
        got = native_mul(Operand.from_poly(a), Operand.from_poly(b), lay, path="bucket")
        want = O.mul(a, b)
        assert got.path == "bucket"
        assert got.exps.tolist() == want.exps
        if ctype is int:
            from paper_1303_7425_b200.parmul import limbs_to_ints
            assert limbs_to_ints(got.coef, got.nl) == want.coeffs
        else:
            assert np.allclose(got.coef, np.asarray(want.coeffs), rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("path", ["auto", "dense", "bucket", "sort", "small"])
def test_degenerate_shapes_and_field_limits(path):
    """1xN, Nx1 and 1x1 products, exponents exactly at the field caps (the
    reference's overflow test is componentwise max <= cap, core.py:365-385),
    and a one-variable lex layout with a 63-bit field, on every path."""
    from paper_1303_7425_b200.core import Layout, VarTable, naive_mul
    lay = default_layout(("x", "y", "z"))
    big = Polynomial(lay, [(k + 1, (k % 7, k % 5, k % 3)) for k in range(300)], int)
    one = Polynomial(lay, [(-3, (2, 0, 1))], int)
    cases = [(big, one), (one, big), (one, one)]
    m = lay.max_total_degree() // 2  # products reach the degree cap exactly
    hi = Polynomial(lay, [(5, (m, 0, 0)), (7, (0, m, 0))], int)
    lo = Polynomial(lay, [(2, (0, 0, 0)), (1, (m, 0, 0)), (-4, (0, 0, m))], int)
    cases.append((hi, lo))
    lex1 = Layout(VarTable(("x",)), "lex", (63,))
    a = Polynomial(lex1, [(1, (0,)), (2, (1 << 40,)), (3, (1 << 61,))], int)
    b = Polynomial(lex1, [(4, (5,)), (-5, (1 << 60,))], int)
    cases.append((a, b))
    for f, g in cases:
        try:
            got = mul(f, g, MulConfig(path=path))
        except Exception as exc:  # the dense path refuses key spans it cannot map
            assert path == "dense" and "dense path" in str(exc)
            continue
        want = naive_mul(f, g)
        assert got.exps == want.exps and got.coeffs == want.coeffs
    with pytest.raises(ExponentOverflowError):
        mul(hi, Polynomial(lay, [(1, (m + 1, 0, 0))], int), MulConfig(path=path))


def test_small_path_is_taken_and_exact(rng):
    """Products of at most 16384 pairs run in one CTA (path_used 'small') and
    equal the oracle, floats bit for bit in the reference's row order."""
    from oracle import oracle as O
    from paper_1303_7425_b200.core import Polynomial as P
    lay = default_layout(("x", "y", "z"))
    for ctype in (int, float):
        for na, nb in [(1, 1), (3, 50), (90, 91), (64, 128)]:
            terms = lambda n: [((rng.randint(-99, 99) or 1) if ctype is int else rng.uniform(-2, 2),
                                tuple(rng.randint(0, 6) for _ in range(3))) for _ in range(n)]
            a, b = P(lay, terms(na), ctype), P(lay, terms(nb), ctype)
            raw = native_mul(Operand.from_poly(a), Operand.from_poly(b), lay)
            assert raw.path == "small" and raw.pairs == a.n * b.n
            want = O.mul(a, b)
            assert raw.exps.tolist() == want.exps
            if ctype is float:
                assert raw.coef.tolist() == want.coeffs  # reference order: bit-identical
            else:
                from paper_1303_7425_b200.parmul import limbs_to_ints
                assert limbs_to_ints(raw.coef, raw.nl) == want.coeffs


def test_concurrent_callers_share_the_device():
    """Several host threads multiplying on the same GPU at once (ctypes drops
    the GIL; the library serialises products per device): every result exact."""
    import threading
    prods = [benchpolys.fateman(6), benchpolys.monagan_pearce(4), benchpolys.fateman(3)]
    want = [mul(f, g) for f, g in prods]
    errors = []

    def worker(k):
        try:
            for r in range(12):
                f, g = prods[(k + r) % len(prods)]
                p = mul(f, g, MulConfig(path=("auto", "sort", "bucket")[(k + r) % 3]))
                w = want[(k + r) % len(prods)]
                if p.exps != w.exps or p.coeffs != w.coeffs:
                    errors.append((k, r))
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_golden_cases_sort_path_column_records(case, monkeypatch):
    """The sort path's 8-byte records (key, column j; the row recovered through
    the hash of operand a's keys), forced on every golden case."""
    monkeypatch.setenv("PGPU_JREC_MIN", "1")
    name, a, b, split, want = case
    got = mul(a, b, MulConfig(path="sort", float_ordered=True), split=None if split is None else SplitSet(split))
    _check(got, want)


@pytest.mark.parametrize("shape", ["one_run", "no_runs", "mixed"])
def test_dense_symbolic_run_intervals_vs_oracle(shape, rng):
    """The dense path's sumset is a union of (a-run x b-run) key intervals
    (dense_path.cuh D1).  Operands made of one long run (runs far wider than a
    window), of isolated keys (one interval per pair) and of mixed run
    lengths, whole and restricted to consecutive packed ranges, against the
    oracle (exact ints)."""
    from oracle import oracle as O
    from paper_1303_7425_b200.core import Polynomial as P
    from paper_1303_7425_b200.parmul import limbs_to_ints
    lay = default_layout(("x", "y"))

    def exps(n, top):
        if shape == "one_run":
            return [(0, e) for e in range(n)]
        if shape == "no_runs":
            return [(0, 2 * e) for e in range(n)]
        pool = sorted(rng.sample(range(top), n))
        return [(e // 64, e % 64) for e in pool]

    def poly(n, top):
        return P(lay, [(rng.randint(-10 ** 9, 10 ** 9), e) for e in exps(n, top)], int)

    a, b = poly(3000, 9000), poly(2500, 9000)
    want = O.mul(a, b)
    A, B = Operand.from_poly(a), Operand.from_poly(b)
    got = native_mul(A, B, lay, path="dense")
    assert got.path == "dense"
    assert got.exps.tolist() == want.exps
    assert limbs_to_ints(got.coef, got.nl) == want.coeffs
    bounds = select_grid(a, b, GridParams(7)).bounds
    cuts = [0] + bounds[1:-1:2] + [(1 << 64) - 1]
    parts = [native_mul(A, B, lay, lo=lo, hi=hi, path="dense") for lo, hi in zip(cuts, cuts[1:])]
    assert np.array_equal(np.concatenate([p.exps for p in parts]), got.exps)
    assert np.array_equal(np.concatenate([p.coef for p in parts]), got.coef)


def test_dense_matches_sort_on_random_dense_products(rng):
    """Twenty random dense-shaped products (2-5 variables, operands cut from
    total-degree simplices with random holes, so run lengths vary from one to
    the full last-field range): the dense path (run-interval sumset, per-warp
    accumulators) equals the sort path bit for bit, whole and on a random
    packed range."""
    from itertools import product as iproduct

    from paper_1303_7425_b200.core import Polynomial as P
    for trial in range(20):
        nv = rng.randint(2, 5)
        lay = default_layout(tuple(f"v{k}" for k in range(nv)))
        deg = {2: 60, 3: 18, 4: 9, 5: 6}[nv]

        def poly():
            keep = rng.uniform(0.3, 1.0)
            terms = [(rng.randint(-10 ** 12, 10 ** 12), e) for e in iproduct(range(deg + 1), repeat=nv)
                     if sum(e) <= deg and rng.random() < keep]
            return P(lay, terms or [(1, (0,) * nv)], int)

        a, b = poly(), poly()
        A, B = Operand.from_poly(a), Operand.from_poly(b)
        d = native_mul(A, B, lay, path="dense")
        s = native_mul(A, B, lay, path="sort")
        assert d.path == "dense", trial
        assert np.array_equal(d.exps, s.exps) and np.array_equal(d.coef, s.coef), trial
        lo, hi = sorted(rng.sample(sorted(set(int(x) for x in s.exps.tolist())) + [0, (1 << 64) - 1], 2))
        dr = native_mul(A, B, lay, lo=lo, hi=hi, path="dense")
        sr = native_mul(A, B, lay, lo=lo, hi=hi, path="sort")
        assert np.array_equal(dr.exps, sr.exps) and np.array_equal(dr.coef, sr.coef), trial
