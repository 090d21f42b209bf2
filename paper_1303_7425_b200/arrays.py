"""Array-backed polynomials: SURVEY 8(f) row 2, the data format downstream of
the hot path.

The reference keeps every polynomial as two Python lists
(`Polynomial._from_sorted`, reference core.py:231-241) and renders results
with `format_poly` (io.py:241-248).  For large products (MP n=25: 3.1e8 terms)
building 3.1e8 Python ints dominates end-to-end time once the product itself
takes a second.  `ArrayPolynomial` keeps the product as the arrays the C ABI
returns -- packed u64 exponents plus f64 coefficients or 1-3 u64 limbs of
two's complement -- and materialises lists only on demand.  It can be fed
back into `mul` (no list round trip) and written as PolyFile text by the GPU
formatter (`io.write_poly`, `pgpu_format`).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .core import CoefficientOverflowError, Polynomial, max_degrees_of

_M64 = (1 << 64) - 1


def int_limbs(coeffs, nl: int | None = None) -> tuple:
    """Python ints -> ((n, nl) u64 two's-complement limbs, nl); nl picked as
    the narrowest of 1..3 limbs that holds every value unless given."""
    if nl is None:
        try:
            return np.asarray(coeffs, dtype=np.int64).view(np.uint64).reshape(-1, 1), 1
        except OverflowError:
            pass
        top = max((abs(c) for c in coeffs), default=0)
        nl = 2 if top.bit_length() < 127 else 3
    lim = 1 << (64 * nl - 1)
    if coeffs and (max(coeffs) >= lim or min(coeffs) < -lim):
        raise CoefficientOverflowError(f"coefficients do not fit {nl} limbs of two's complement")
    out = np.empty((len(coeffs), nl), dtype=np.uint64)
    for k in range(nl):
        out[:, k] = [(c >> (64 * k)) & _M64 for c in coeffs]
    return out, nl


class ArrayPolynomial:
    """Canonical polynomial held in arrays (same contract as Polynomial:
    strictly ascending exponents, no zero coefficients, one ctype)."""

    __slots__ = ("layout", "ctype", "_exps", "_coef", "nl", "_lists", "_maxes")

    def __init__(self, layout, exps: np.ndarray, coef: np.ndarray, ctype: type = int, nl: int = 1):
        self.layout = layout
        self.ctype = ctype
        self._exps = np.ascontiguousarray(exps, dtype=np.uint64)
        if ctype is float:
            self._coef = np.ascontiguousarray(coef, dtype=np.float64).reshape(-1)
            self.nl = 1
        else:
            self._coef = np.ascontiguousarray(coef).view(np.uint64).reshape(-1, nl)
            self.nl = nl
        if self._coef.shape[0] != self._exps.shape[0]:
            raise ValueError("exponent and coefficient arrays differ in length")
        self._lists = None
        self._maxes = None

    # -- construction ------------------------------------------------------
    @classmethod
    def from_poly(cls, p) -> "ArrayPolynomial":
        if isinstance(p, ArrayPolynomial):
            return p
        exps = p.exps_array() if hasattr(p, "exps_array") else np.fromiter(p.exps, np.uint64, len(p.exps))
        if p.ctype is float:
            return cls(p.layout, exps, np.asarray(p.coeffs, dtype=np.float64), float)
        limbs, nl = int_limbs(list(p.coeffs))
        return cls(p.layout, exps, limbs, int, nl)

    @classmethod
    def from_raw(cls, layout, ctype, raw) -> "ArrayPolynomial":
        """From a parmul.RawProduct (arrays straight from the C ABI)."""
        if ctype is float:
            return cls(layout, raw.exps, raw.coef, float)
        return cls(layout, raw.exps, raw.coef, int, raw.nl)

    @classmethod
    def _from_sorted(cls, layout, exps: list, coeffs: list, ctype: type = int) -> "ArrayPolynomial":
        return cls.from_poly(Polynomial._from_sorted(layout, exps, coeffs, ctype))

    @classmethod
    def zero(cls, layout, ctype: type = int) -> "ArrayPolynomial":
        coef = np.zeros(0, np.float64) if ctype is float else np.zeros((0, 1), np.uint64)
        return cls(layout, np.zeros(0, np.uint64), coef, ctype)

    # -- the Polynomial surface ---------------------------------------------
    @property
    def n(self) -> int:
        return int(self._exps.shape[0])

    def __len__(self):
        return self.n

    @property
    def is_zero(self) -> bool:
        return self.n == 0

    def exps_array(self) -> np.ndarray:
        return self._exps

    def coef_array(self) -> np.ndarray:
        """float64 (n,) or u64 (n, nl) limbs."""
        return self._coef

    def _materialise(self):
        if self._lists is None:
            from .parmul import limbs_to_ints
            exps = self._exps.tolist()
            coeffs = self._coef.tolist() if self.ctype is float else limbs_to_ints(self._coef, self.nl)
            self._lists = (exps, coeffs)
        return self._lists

    @property
    def exps(self) -> list:
        return self._materialise()[0]

    @property
    def coeffs(self) -> list:
        return self._materialise()[1]

    def terms(self):
        return zip(self.coeffs, self.exps)

    def terms_vec(self):
        up = self.layout.unpack
        return ((c, up(e)) for c, e in zip(self.coeffs, self.exps))

    def max_degrees(self) -> tuple:
        if self._maxes is None:
            self._maxes = max_degrees_of(self)
        return self._maxes

    def to_poly(self, cls=Polynomial):
        exps, coeffs = self._materialise()
        return cls._from_sorted(self.layout, exps, coeffs, self.ctype)

    def __eq__(self, other):
        if not hasattr(other, "layout") or not hasattr(other, "ctype"):
            return NotImplemented
        if not (self.layout == other.layout and self.ctype is other.ctype and self.n == other.n):
            return False
        oe = other.exps_array() if hasattr(other, "exps_array") else np.fromiter(other.exps, np.uint64, other.n)
        if not np.array_equal(self._exps, oe):
            return False
        return self.coeffs == list(other.coeffs)

    __hash__ = None

    def __mul__(self, other):
        from .parmul import mul
        return mul(self, other)

    def __repr__(self):
        kind = "int" if self.ctype is int else "f64"
        return (f"<ArrayPolynomial {self.n} terms over "
                f"{','.join(self.layout.vars.names)} ({self.layout.order}, {kind}, {self.nl} limb(s))>")

    # -- C-ABI views ---------------------------------------------------------
    def operand(self):
        """parmul.Operand without a list round trip (ints narrowed to the
        operand widths the ABI accepts: int64 or two limbs)."""
        from .parmul import Operand
        if self.ctype is float:
            return Operand(self._exps, self._coef, N.F64)
        c = self._coef
        sign = (c[:, -1].view(np.int64) >> 63).view(np.uint64)

        def fits(width: int) -> bool:  # two's complement value fits `width` limbs
            if width >= self.nl:
                return True
            return (all(np.array_equal(c[:, k], sign) for k in range(width, self.nl))
                    and np.array_equal((c[:, width - 1].view(np.int64) >> 63).view(np.uint64), sign))

        if fits(1):
            return Operand(self._exps, np.ascontiguousarray(c[:, 0]).view(np.int64), N.I64)
        if fits(2):
            return Operand(self._exps, np.ascontiguousarray(c[:, :2]), N.I128)
        raise CoefficientOverflowError(
            "operand coefficients beyond 127 bits are not supported by the GPU path")
