"""The PolyFile formatter (csrc/text.cuh) compiled for the
host with g++ and checked against Python's own str(int) / repr(float) -- the
functions the reference's format_poly calls (io.py:241-248) -- plus the
host logic of ArrayPolynomial.  No GPU needed; the device build of the same
code is checked in tests/test_gpu_format.py."""

from __future__ import annotations

import ctypes as C
import random
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import golden_cases
from paper_1303_7425_b200 import io
from paper_1303_7425_b200.arrays import ArrayPolynomial, int_limbs
from paper_1303_7425_b200.core import CoefficientOverflowError, Polynomial, _fields_of, default_layout
from paper_1303_7425_b200 import _native as N

SRC = Path(__file__).resolve().parent / "native" / "fmt_host.cpp"


class LineSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("nl", C.c_int), ("nvars", C.c_int),
                ("shift", C.c_int * 15), ("mask", C.c_uint64 * 15)]


@pytest.fixture(scope="module")
def fmt(tmp_path_factory):
    so = tmp_path_factory.mktemp("fmt") / "fmt_host.so"
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-std=c++17", "-o", str(so), str(SRC)], check=True)
    lib = C.CDLL(str(so))
    lib.fmt_doubles.argtypes = [C.c_void_p, C.c_int64, C.c_char_p]
    lib.fmt_doubles.restype = C.c_int64
    lib.fmt_ints.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_char_p]
    lib.fmt_ints.restype = C.c_int64
    lib.fmt_lines.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(LineSpec), C.c_char_p]
    lib.fmt_lines.restype = C.c_int64
    return lib


def doubles_text(lib, vals) -> list:
    v = np.ascontiguousarray(vals, dtype=np.float64)
    buf = C.create_string_buffer(v.size * 32 + 16)
    n = lib.fmt_doubles(v.ctypes.data, v.size, buf)
    assert n >= 0, f"count/write disagree at {-1 - n}"
    return buf.raw[:n].decode().split("\n")[:-1]


def check_doubles(lib, vals):
    v = np.ascontiguousarray(vals, dtype=np.float64)
    got = doubles_text(lib, v)
    want = [repr(x) for x in v.tolist()]
    bad = [(w, g) for w, g in zip(want, got) if w != g]
    assert not bad, bad[:5]


def test_repr_random_bit_patterns(fmt):
    rng = np.random.default_rng(0x7E47)
    bits = rng.integers(0, 2 ** 63, size=300_000, dtype=np.int64).view(np.uint64)
    bits |= rng.integers(0, 2, size=bits.size, dtype=np.uint64) << np.uint64(63)
    check_doubles(fmt, bits.view(np.float64))


def test_repr_decimal_boundaries(fmt):
    vals = []
    for k in range(-30, 40):
        b = struct.unpack("<Q", struct.pack("<d", 10.0 ** k))[0]
        vals += [struct.unpack("<d", struct.pack("<Q", b + d))[0] for d in range(-40, 40)]
    vals += [float(10 ** k) for k in range(309)] + [2.0 ** k for k in range(-1074, 1024)]
    vals += [x * 0.1 for x in range(-5000, 5000)] + [float(x) for x in range(-3000, 3000)]
    vals += [1e16, 1e15, 123456789012345680.0, 1234567890123456.0, 0.0001, 0.00001, 1e-5, 9.999e-5]
    check_doubles(fmt, vals)


def test_repr_subnormals_and_specials(fmt):
    check_doubles(fmt, np.arange(1, 20000, dtype=np.uint64).view(np.float64))
    check_doubles(fmt, [5e-324, 2.2250738585072014e-308, 2.225073858507201e-308,
                        1.7976931348623157e308, float("inf"), float("-inf"), 0.0, -0.0,
                        0.1, 0.2, 0.3, 1 / 3, 2 / 3, 9007199254740993.0, 1e22, 1e23])
    assert doubles_text(fmt, [float("nan")]) == ["nan"]


@pytest.mark.parametrize("nl", [1, 2, 3])
def test_str_of_limbed_ints(fmt, nl):
    R = random.Random(nl)
    B = 64 * nl
    vals = [R.randrange(-2 ** (B - 1), 2 ** (B - 1)) >> R.randrange(0, B) for _ in range(50_000)]
    vals += [0, 1, -1, 2 ** (B - 1) - 1, -2 ** (B - 1), 999999999, 1000000000, -1000000000]
    vals += [10 ** k for k in range(int(B * 0.301))] + [1 - 10 ** k for k in range(int(B * 0.301))]
    arr, _ = int_limbs(vals, nl)
    buf = C.create_string_buffer(len(vals) * 64 + 16)
    n = fmt.fmt_ints(arr.ctypes.data, nl, len(vals), buf)
    assert n >= 0
    got = buf.raw[:n].decode().split("\n")[:-1]
    assert got == [str(v) for v in vals]


def line_spec(layout, kind, nl) -> LineSpec:
    fl = _fields_of(layout)
    first = 1 if layout.order == "grlex" else 0
    s = LineSpec()
    s.kind, s.nl, s.nvars = kind, nl, len(fl) - first
    for k, (sh, w) in enumerate(fl[first:]):
        s.shift[k] = sh
        s.mask[k] = (1 << w) - 1 if w < 64 else (1 << 64) - 1
    return s


CASES = golden_cases()


@pytest.mark.parametrize("case", CASES[::3], ids=[c[0] for c in CASES[::3]])
def test_lines_match_format_poly(fmt, case):
    """Whole PolyFile lines of the golden operands (ints up to 2^90 and 3^60,
    inf/nan floats, lex and 14-variable layouts) equal format_poly's."""
    _, a, b, _, _ = case
    for p in (a, b):
        exps, coef, kind, nl = io._arrays(p)
        spec = line_spec(p.layout, 0 if kind == N.F64 else 1, nl)
        buf = C.create_string_buffer(max(1, p.n) * 512)
        n = fmt.fmt_lines(exps.ctypes.data, coef.ctypes.data, p.n, C.byref(spec), buf)
        text = io.header(p.layout).decode() + buf.raw[:n].decode()
        assert text == io.format_poly(p)


def test_array_polynomial_round_trip_and_equality():
    lay = default_layout(("x", "y"))
    p = Polynomial(lay, [(3, (1, 0)), (-(2 ** 100), (0, 2)), (7, (0, 0))], int)
    ap = ArrayPolynomial.from_poly(p)
    assert ap.nl == 2 and ap.n == 3 and ap == p and ap.to_poly() == p
    assert ap.exps == p.exps and ap.coeffs == p.coeffs
    assert ap.max_degrees() == p.max_degrees()
    op = ap.operand()
    assert op.kind == N.I128 and op.coef.shape == (3, 2)
    small = ArrayPolynomial.from_poly(Polynomial(lay, [(5, (1, 1)), (-4, (0, 0))], int))
    assert small.operand().kind == N.I64
    wide = ArrayPolynomial(lay, p.exps_array(), int_limbs(p.coeffs, 3)[0], int, 3)
    assert wide == p and wide.operand().kind == N.I128  # narrowed back to two limbs
    huge = ArrayPolynomial.from_poly(Polynomial(lay, [(2 ** 150, (1, 0))], int))
    assert huge.nl == 3
    with pytest.raises(CoefficientOverflowError):
        huge.operand()
    fp = Polynomial(lay, [(0.5, (1, 0)), (float("inf"), (0, 0))], float)
    fa = ArrayPolynomial.from_poly(fp)
    assert fa == fp and fa.operand().kind == N.F64
    assert ArrayPolynomial.zero(lay).is_zero
