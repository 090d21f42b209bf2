"""PolyFile text writer (reference io.py:241-248), used as the golden-digest
serializer: sha256(format_poly(product)) is the parity fingerprint recorded
from the reference."""

from __future__ import annotations

import hashlib


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
