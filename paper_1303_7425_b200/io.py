"""PolyFile text (reference io.py:241-248 `format_poly`, io.py:306-308
`write_poly`): SURVEY 8(f) row 2, the on-disk format downstream of the
product.

`format_poly` / `poly_digest` here are the plain host serializers used as
the golden-digest fingerprint (sha256 of the reference's format_poly,
SURVEY.md Appendix A).  `format_text` / `write_poly` / `text_digest` are the
product path: the term lines are formatted on the GPU by `pgpu_format`
(csrc/format.cuh; integers as str(), doubles as repr()) in bounded chunks,
straight from the product's arrays -- no Python int or float is created.
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np

from . import _native as N

DEFAULT_CHUNK_TERMS = 1 << 22
_FLOAT_MARKS = (".", "e", "E", "n", "i")  # decimals, exponents, nan/inf


class PolyIOError(ValueError):
    """Malformed polynomial file; the message names the offending line
    (reference io.py:34-35)."""


def parse_poly(text: str, layout=None, ctype=None):
    """PolyFile text -> Polynomial (reference io.py:251-290, same rules and
    messages): a `vars` header, then `coeff e1 ... em` lines; '#' comments and
    blank lines skipped; duplicate exponents combined; ctype inferred from the
    coefficient spelling unless given.  Host-side input parsing (operands)."""
    from .core import Polynomial, VarTable, default_layout
    vars_decl = None
    raw = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        st = line.strip()
        if not st or st.startswith("#"):
            continue
        fields = st.split()
        if vars_decl is None:
            if fields[0] != "vars" or len(fields) < 2:
                raise PolyIOError(f"line {lineno}: expected 'vars <name>...' header")
            try:
                vars_decl = VarTable(tuple(fields[1:]))
            except ValueError as exc:
                raise PolyIOError(f"line {lineno}: {exc}") from None
            continue
        raw.append((lineno, fields))
    if vars_decl is None:
        raise PolyIOError("missing 'vars' header line")
    if layout is None:
        layout = default_layout(vars_decl.names)
    elif tuple(layout.vars.names) != tuple(vars_decl.names):
        raise PolyIOError(f"file declares variables {vars_decl.names}, expected {layout.vars.names}")
    if ctype is None:
        ctype = float if any(any(m in f[0] for m in _FLOAT_MARKS) for _, f in raw) else int
    terms = []
    for lineno, fields in raw:
        if len(fields) != 1 + vars_decl.m:
            raise PolyIOError(f"line {lineno}: expected coefficient plus {vars_decl.m} exponents, "
                              f"got {len(fields)} fields")
        try:
            coeff = ctype(fields[0])
            vec = tuple(int(f) for f in fields[1:])
        except ValueError:
            raise PolyIOError(f"line {lineno}: malformed number") from None
        if any(v < 0 for v in vec):
            raise PolyIOError(f"line {lineno}: negative exponent")
        terms.append((coeff, vec))
    return Polynomial(layout, terms, ctype)


def read_poly(path, layout=None, ctype=None):
    """reference io.read_poly (io.py:301-303)."""
    with open(path, "r", encoding="utf-8") as fh:
        return parse_poly(fh.read(), layout, ctype)


def format_poly(poly) -> str:
    """`vars x y ...` header, then one `coeff e1 ... em` line per term,
    ascending; floats in repr() form so they round-trip."""
    head = "vars " + " ".join(poly.layout.vars.names)
    show = repr if poly.ctype is float else str
    up = poly.layout.unpack
    body = [show(c) + " " + " ".join(map(str, up(e))) for c, e in zip(poly.coeffs, poly.exps)]
    return "\n".join([head] + body) + "\n"


def poly_digest(poly) -> str:
    return hashlib.sha256(format_poly(poly).encode()).hexdigest()


# ---------------------------------------------------------------------------
# GPU formatter
# ---------------------------------------------------------------------------
def header(layout) -> bytes:
    return ("vars " + " ".join(layout.vars.names) + "\n").encode()


def _arrays(p):
    """(exps u64, coefficient array, coef_kind, limbs) of a Polynomial or
    ArrayPolynomial, without building Python objects for ArrayPolynomial."""
    from .arrays import ArrayPolynomial
    ap = p if isinstance(p, ArrayPolynomial) else ArrayPolynomial.from_poly(p)
    if ap.ctype is float:
        return ap.exps_array(), ap.coef_array(), N.F64, 1
    return ap.exps_array(), ap.coef_array(), N.I64, ap.nl


def format_terms(exps: np.ndarray, coef: np.ndarray, kind: int, nl: int, layout,
                 begin: int = 0, end: int | None = None, device: int = 0) -> bytes:
    """Term lines [begin, end) of host arrays through pgpu_format."""
    n = int(exps.shape[0])
    end = n if end is None else end
    if end <= begin:
        return b""
    lib = N.load()
    exps = np.ascontiguousarray(exps, dtype=np.uint64)
    coef = np.ascontiguousarray(coef)
    poly = N.Poly(exps.ctypes.data, coef.ctypes.data, n)
    o = N.default_options()
    o.coef_kind = kind
    o.acc_limbs = nl
    o.device = device
    lay = N.make_layout(layout)
    t = N.Text()
    st = lib.pgpu_format(C.byref(poly), C.byref(lay), begin, end, C.byref(o), C.byref(t))
    if st != N.PGPU_OK:
        from .parmul import _raise_status
        _raise_status(st)
    try:
        return C.string_at(t.text, t.bytes) if t.bytes else b""
    finally:
        lib.pgpu_free_text(C.byref(t))


def format_device(res, layout, begin: int = 0, end: int | None = None, device: int = 0) -> bytes:
    """Term lines of a device-resident product (device.DeviceResult): the
    formatter reads the result where the multiplier left it."""
    end = res.n if end is None else end
    if end <= begin:
        return b""
    lib = N.load()
    poly = N.Poly(res.res.exps, res.res.coeffs, res.n)
    o = N.default_options()
    o.coef_kind = res.kind
    o.acc_limbs = res.nl
    o.device = device
    o.inputs_on_device = 1
    lay = N.make_layout(layout)
    t = N.Text()
    st = lib.pgpu_format(C.byref(poly), C.byref(lay), begin, end, C.byref(o), C.byref(t))
    if st != N.PGPU_OK:
        from .parmul import _raise_status
        _raise_status(st)
    try:
        return C.string_at(t.text, t.bytes) if t.bytes else b""
    finally:
        lib.pgpu_free_text(C.byref(t))


def iter_text(p, chunk_terms: int = DEFAULT_CHUNK_TERMS, device: int = 0):
    """PolyFile bytes of p: the header, then the term lines in chunks of at
    most chunk_terms terms (bounded host and device memory for any size)."""
    exps, coef, kind, nl = _arrays(p)
    yield header(p.layout)
    n = int(exps.shape[0])
    for b in range(0, n, chunk_terms):
        yield format_terms(exps, coef, kind, nl, p.layout, b, min(n, b + chunk_terms), device)


def format_text(p, device: int = 0) -> str:
    """GPU-formatted equivalent of format_poly(p)."""
    return b"".join(iter_text(p, device=device)).decode()


def write_poly(path, p, device: int = 0, chunk_terms: int = DEFAULT_CHUNK_TERMS) -> int:
    """reference io.write_poly (io.py:306-308) with GPU formatting; returns bytes written."""
    total = 0
    with open(path, "wb") as fh:
        for part in iter_text(p, chunk_terms, device):
            fh.write(part)
            total += len(part)
    return total


def text_digest(p, device: int = 0, chunk_terms: int = DEFAULT_CHUNK_TERMS) -> str:
    """sha256 of format_poly(p), formatted on the GPU chunk by chunk."""
    h = hashlib.sha256()
    for part in iter_text(p, chunk_terms, device):
        h.update(part)
    return h.hexdigest()
