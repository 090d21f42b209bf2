"""GPU PolyFile formatter and array-backed products.

The text pgpu_format produces must equal the reference's format_poly
(io.py:241-248) byte for byte: checked on every golden product and against
the reference's sha256 digests of format_poly(mul(f, g)) for the benchmark
configurations, with products kept as arrays
(mul_arrays) so no Python int or float is built on the way."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import digests, golden_cases
from paper_1303_7425_b200 import MulConfig, Polynomial, benchpolys, default_layout, io, mul
from paper_1303_7425_b200.arrays import ArrayPolynomial, int_limbs
from paper_1303_7425_b200.parmul import Operand, mul_arrays
from paper_1303_7425_b200.split import SplitSet

pytestmark = pytest.mark.gpu
CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_golden_products_format_like_format_poly(case):
    _, a, b, split, _ = case
    p = mul_arrays(a, b, MulConfig(float_ordered=True), split=None if split is None else SplitSet(split))
    ref = mul(a, b, MulConfig(float_ordered=True), split=None if split is None else SplitSet(split))
    want = io.format_poly(ref)  # (text, not ==: nan coefficients never compare equal)
    assert io.format_poly(p.to_poly()) == want
    assert io.format_text(p) == want
    for op in (a, b):  # operands too: Python ints of any width up to 191 bits
        assert io.format_text(op) == io.format_poly(op)


@pytest.mark.parametrize("cfg", ["fateman10/int", "fateman20/int", "fateman30/int", "mp12/int",
                                 "fateman10/float"])
def test_reference_digests_from_gpu_text(cfg):
    name, kind = cfg.split("/")
    f, g = benchpolys.CONFIGS[name](float if kind == "float" else int)
    p = mul_arrays(f, g)
    want = digests()["products"][cfg]
    assert p.n == want["n"]
    assert io.text_digest(p) == want["sha256"]


@pytest.mark.parametrize("cfg", ["fateman20/float", "mp12/float"])
def test_reference_float_digests_from_gpu_text(cfg):
    name, _ = cfg.split("/")
    f, g = benchpolys.CONFIGS[name](float)
    p = mul_arrays(f, g, MulConfig(float_ordered=True))
    want = digests()["products"][cfg]
    assert p.n == want["n"] and io.text_digest(p) == want["sha256"]


def test_chunking_and_file_writer(tmp_path):
    f, g = benchpolys.CONFIGS["fateman20"](int)
    p = mul_arrays(f, g)
    want = digests()["products"]["fateman20/int"]["sha256"]
    assert io.text_digest(p, chunk_terms=9973) == want
    path = tmp_path / "f20.poly"
    nbytes = io.write_poly(path, p, chunk_terms=50_000)
    data = path.read_bytes()
    assert len(data) == nbytes
    import hashlib
    assert hashlib.sha256(data).hexdigest() == want


def test_device_resident_result_formats_in_place():
    from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
    import torch
    f, g = benchpolys.CONFIGS["mp12"](int)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    dev = torch.device("cuda", 0)
    res = mul_on_device(DeviceOperand(A, dev), DeviceOperand(B, dev), f.layout)
    try:
        text = io.header(f.layout) + io.format_device(res, f.layout)
    finally:
        res.free()
    import hashlib
    assert hashlib.sha256(text).hexdigest() == digests()["products"]["mp12/int"]["sha256"]


def test_array_products_chain_without_lists():
    """Powering with ArrayPolynomial operands (the eval_expr caller, 8(f)
    row 1) gives the same polynomial as the list-based path."""
    lay = default_layout(("x", "y", "z", "t"))
    from paper_1303_7425_b200.expr import poly_from_expr
    base = poly_from_expr("1+x+y+z+t", lay)
    ap = ArrayPolynomial.from_poly(base)
    acc = ap
    for _ in range(4):
        acc = mul_arrays(acc, acc)  # (1+x+y+z+t)^16, coefficients up to 16!/4!^4
    assert isinstance(acc, ArrayPolynomial)
    assert acc == poly_from_expr("(1+x+y+z+t)^16", lay)


def test_wide_integer_text():
    lay = default_layout(("x", "y"))
    vals = [2 ** 190 - 1, -(2 ** 190), 3 ** 100, -(3 ** 99), 1, -1, 10 ** 57]
    p = Polynomial(lay, [(c, (k, 0)) for k, c in enumerate(vals)], int)
    assert io.format_text(p) == io.format_poly(p)
    limbs, nl = int_limbs(p.coeffs)
    assert nl == 3
    ap = ArrayPolynomial(lay, p.exps_array(), limbs, int, nl)
    assert io.format_text(ap) == io.format_poly(p)
