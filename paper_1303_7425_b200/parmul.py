"""Drop-in replacement for the reference hot path `polymul.parmul.mul`.

    mul(a, b, cfg=None, *, split=None) -> Polynomial        (parmul.py:91-109)

Host side does exactly what the reference does before its merge loop --
compatibility check (core.py:333-337), zero short-circuit (parmul.py:102-103),
exponent-fit check (core.py:365-385) -- then marshals both operands into flat
arrays and runs the whole product on the GPU through the C ABI
(include/polymul_b200.h).  The result is rebuilt with the operand class's own
`_from_sorted`, so reference `polymul.core.Polynomial` objects go in and come
out unchanged in type.

`cfg.l` (grid density) and `cfg.c` (worker count) keep their reference meaning
for the multi-GPU split (`cluster.gpu_mul`); on one GPU the device picks its
own interval geometry, which never changes the result (split.py:1-9: any
covering split gives the same product).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import (SENTINEL, CoefficientOverflowError, ExponentOverflowError, check_compatible,
                   check_product_fits)

MERGERS = ("heap", "tree")
PATHS = {"auto": N.PATH_AUTO, "dense": N.PATH_DENSE, "sort": N.PATH_SORT, "bucket": N.PATH_BUCKET,
         "small": N.PATH_SMALL}
PATH_NAMES = {1: "dense", 2: "sort", 3: "bucket", 4: "small"}
DEFAULT_GRID_DENSITY = 64
_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class MulConfig:
    """Reference knobs (parmul.py:29-43) plus GPU selections.

    l, c, merger  -- as in the reference; `merger` names the CPU merge the
                     reference would use and is validated the same way; both
                     produce identical output (merge.py:1-16), as does the GPU.
    path          -- "auto" | "dense" | "sort" | "bucket" | "small" (device algorithm)
    float_ordered -- float coefficients: True folds every term in the
                     reference's row order (merge.py:32-33), so doubles are
                     bit-identical to the CPU (the dense path is skipped);
                     False also allows the dense path, whose warp copies fold
                     a term in a fixed order of its own (run-to-run identical,
                     within 2k*2^-53*sum|a_i b_j| of the reference); None
                     (default) means True
    device        -- CUDA ordinal
    """

    l: int = DEFAULT_GRID_DENSITY
    c: int = 1
    merger: str = "heap"
    path: str = "auto"
    float_ordered: bool | None = None
    device: int = 0

    @property
    def ordered(self) -> bool:
        return self.float_ordered is None or bool(self.float_ordered)

    @classmethod
    def of(cls, cfg) -> "MulConfig":
        """Our config from None, our own, or the reference's MulConfig (l, c,
        merger; parmul.py:29-43) -- the drop-in receives the reference's."""
        if cfg is None:
            return cls()
        if isinstance(cfg, cls):
            return cfg
        return cls(l=getattr(cfg, "l", DEFAULT_GRID_DENSITY), c=getattr(cfg, "c", 1),
                   merger=getattr(cfg, "merger", "heap"), path=getattr(cfg, "path", "auto"),
                   float_ordered=getattr(cfg, "float_ordered", None), device=getattr(cfg, "device", 0))

    def __post_init__(self):
        if self.l < 1:
            raise ValueError(f"grid density must be >= 1, got {self.l}")
        if self.c < 1:
            raise ValueError(f"worker count must be >= 1, got {self.c}")
        if self.merger not in MERGERS:
            raise ValueError(f"merger must be one of {sorted(MERGERS)}, got {self.merger!r}")
        if self.path not in PATHS:
            raise ValueError(f"path must be one of {sorted(PATHS)}, got {self.path!r}")


# ---------------------------------------------------------------------------
# Operand marshaling
# ---------------------------------------------------------------------------
class Operand:
    """Flat host arrays of one polynomial, ready for the C ABI."""

    __slots__ = ("exps", "coef", "kind", "n")

    def __init__(self, exps: np.ndarray, coef: np.ndarray, kind: int):
        self.exps = np.ascontiguousarray(exps, dtype=np.uint64)
        self.coef = np.ascontiguousarray(coef)
        self.kind = kind
        self.n = int(self.exps.shape[0])

    @classmethod
    def from_poly(cls, p, kind: int | None = None) -> "Operand":
        if hasattr(p, "operand"):  # ArrayPolynomial: arrays straight through
            return p.operand()
        exps = p.exps_array() if hasattr(p, "exps_array") else np.fromiter(p.exps, np.uint64, len(p.exps))
        if p.ctype is float:
            return cls(exps, np.asarray(p.coeffs, dtype=np.float64), N.F64)
        return cls(exps, *int_coeff_array(p.coeffs, kind))

    def struct(self) -> N.Poly:
        return N.Poly(self.exps.ctypes.data, self.coef.ctypes.data, self.n)


def int_coeff_array(coeffs, kind: int | None = None):
    """Python ints -> (array, kind): int64 when every value fits, else two
    little-endian u64 limbs (two's complement, |c| < 2^127)."""
    if kind in (None, N.I64):
        try:
            return np.asarray(coeffs, dtype=np.int64), N.I64
        except OverflowError:
            if kind == N.I64:
                raise
    out = np.empty((len(coeffs), 2), dtype=np.uint64)
    try:
        out[:, 0] = [c & _M64 for c in coeffs]
        out[:, 1] = np.asarray([c >> 64 for c in coeffs], dtype=np.int64).view(np.uint64)
    except OverflowError:
        raise CoefficientOverflowError(
            "operand coefficients beyond 127 bits are not supported by the GPU path") from None
    return out, N.I128


_PYLIMBS = None


def _pylimbs():
    """The C marshaling helper (csrc/pylimbs.c, lib/_pylimbs*.so), or None."""
    global _PYLIMBS
    if _PYLIMBS is None:
        _PYLIMBS = False
        try:
            import importlib.util
            import sysconfig
            from pathlib import Path
            path = Path(__file__).resolve().parent / "lib" / ("_pylimbs" + sysconfig.get_config_var("EXT_SUFFIX"))
            if path.exists():
                spec = importlib.util.spec_from_file_location("_pylimbs", path)
                mod = importlib.util.module_from_spec(spec)
                spec.loader.exec_module(mod)
                _PYLIMBS = mod
        except Exception:  # marshaling only: the Python conversion below is equivalent
            _PYLIMBS = False
    return _PYLIMBS or None


def limbs_to_ints(limbs: np.ndarray, nl: int) -> list:
    """(n, nl) u64 two's-complement limbs -> Python ints.

    Built in C by the marshaling helper when it is present (about 5x faster);
    otherwise values that fit int64 go through numpy's tolist and the rest
    through int.from_bytes on their little-endian limb bytes."""
    if limbs.size == 0:
        return []
    limbs = np.ascontiguousarray(limbs.reshape(-1, nl))
    helper = _pylimbs()
    if helper is not None:
        return helper.limbs_to_list(memoryview(limbs).cast("B"), limbs.shape[0], nl)
    lo = limbs[:, 0].view(np.int64)
    if nl == 1:
        return lo.tolist()
    sign = (lo >> 63).view(np.uint64)
    small = np.all(limbs[:, 1:] == sign[:, None], axis=1)
    out = lo.tolist()
    idx = np.nonzero(~small)[0]
    if idx.size:
        raw = limbs[idx].tobytes()
        w = 8 * nl
        fb = int.from_bytes
        for t, pos in enumerate(idx.tolist()):
            out[pos] = fb(raw[t * w:(t + 1) * w], "little", signed=True)
    return out


# ---------------------------------------------------------------------------
# Raw product (arrays in, arrays out)
# ---------------------------------------------------------------------------
@dataclass
class RawProduct:
    exps: np.ndarray          # uint64, ascending
    coef: np.ndarray          # float64 (n,) or uint64 (n, nl)
    kind: int                 # F64 or I64 (limbed)
    nl: int
    pairs: int
    path: str
    launches: int
    key_bits: int
    phases: dict


def _raise_status(st: int):
    msg = N.last_error()
    if st == N.PGPU_EEXPONENT:
        raise ExponentOverflowError(msg)
    if st == N.PGPU_ECOEFF:
        raise CoefficientOverflowError(msg)
    if st == N.PGPU_EINVAL:
        raise ValueError(msg)
    raise N.NativeError(f"pgpu status {st}: {msg}")


def native_mul(A: Operand, B: Operand, layout, *, lo: int = 0, hi: int = SENTINEL,
               path: str = "auto", float_ordered: bool = False, device: int = 0,
               timing: bool = False, stream=None) -> RawProduct:
    """One product through pgpu_mul with host buffers (H2D/D2H inside)."""
    if A.kind == N.F64 and B.kind != N.F64 or B.kind == N.F64 and A.kind != N.F64:
        raise ValueError("operands use different coefficient types")
    if A.kind != B.kind:  # widen the int64 side to limbs
        A = A if A.kind == N.I128 else _widen(A)
        B = B if B.kind == N.I128 else _widen(B)
    lib = N.load()
    o = N.default_options()
    o.coef_kind = A.kind
    o.device = device
    o.path = PATHS[path]
    o.float_ordered = int(bool(float_ordered))
    o.timing = int(bool(timing))
    o.lo = lo
    o.hi = hi
    o.stream = stream
    pa, pb = A.struct(), B.struct()
    lay = N.make_layout(layout)
    res = N.Result()
    st = lib.pgpu_mul(C.byref(pa), C.byref(pb), C.byref(lay), C.byref(o), C.byref(res))
    if st != N.PGPU_OK:
        _raise_status(st)
    try:
        n = int(res.n)
        nl = int(res.acc_limbs) or 1
        if n:
            exps = np.ctypeslib.as_array(C.cast(res.exps, C.POINTER(C.c_uint64)), (n,)).copy()
            if res.coef_kind == N.F64:
                coef = np.ctypeslib.as_array(C.cast(res.coeffs, C.POINTER(C.c_double)), (n,)).copy()
            else:
                coef = np.ctypeslib.as_array(C.cast(res.coeffs, C.POINTER(C.c_uint64)), (n * nl,)).copy()
                coef = coef.reshape(n, nl)
        else:
            exps = np.zeros(0, np.uint64)
            coef = np.zeros(0, np.float64) if res.coef_kind == N.F64 else np.zeros((0, nl), np.uint64)
        phases = {}
        for k in range(res.n_phase):
            name = res.phase_name[k]
            phases[name.decode() if name else f"phase{k}"] = float(res.phase_ms[k])
        return RawProduct(exps, coef, int(res.coef_kind), nl, int(res.pairs),
                          PATH_NAMES.get(int(res.path_used), "none"),
                          int(res.kernel_launches), int(res.key_bits), phases)
    finally:
        lib.pgpu_free_result(C.byref(res))


def _widen(op: Operand) -> Operand:
    v = op.coef.astype(np.int64)
    out = np.empty((op.n, 2), dtype=np.uint64)
    out[:, 0] = v.view(np.uint64)
    out[:, 1] = (v >> 63).view(np.uint64)
    return Operand(op.exps, out, N.I128)


# ---------------------------------------------------------------------------
# The drop-in
# ---------------------------------------------------------------------------
def mul(a, b, cfg: MulConfig | None = None, *, split=None):
    """Product of two polynomials over the same variables (parmul.py:91-109).

    Exactly equal to the schoolbook product for int coefficients; for floats
    equal within 2*k*2^-53*sum|a_i b_j| per term (k = products in the term),
    and bit-identical by default (cfg.float_ordered None/True).  `split` keeps the reference's
    semantics: products whose exponent is below split.bounds[0] are not formed
    (split.py:44-50 only checks ascent and the sentinel).
    """
    cfg = MulConfig.of(cfg)
    check_compatible(a, b)
    cls = type(a)
    if a.is_zero or b.is_zero:
        return cls.zero(a.layout, a.ctype)
    check_product_fits(a, b)
    lo = 0
    if split is not None:
        lo = int(split.bounds[0])
    raw = native_mul(Operand.from_poly(a), Operand.from_poly(b), a.layout, lo=lo,
                     path=cfg.path, float_ordered=cfg.ordered, device=cfg.device)
    return to_poly(cls, a.layout, a.ctype, raw)


def mul_arrays(a, b, cfg: MulConfig | None = None, *, split=None):
    """`mul` returning an ArrayPolynomial: the product stays in the arrays
    the C ABI returns; Python lists are built only if
    asked for.  Operands may be Polynomial or ArrayPolynomial."""
    from .arrays import ArrayPolynomial
    cfg = MulConfig.of(cfg)
    check_compatible(a, b)
    if a.is_zero or b.is_zero:
        return ArrayPolynomial.zero(a.layout, a.ctype)
    check_product_fits(a, b)
    lo = 0 if split is None else int(split.bounds[0])
    raw = native_mul(Operand.from_poly(a), Operand.from_poly(b), a.layout, lo=lo,
                     path=cfg.path, float_ordered=cfg.ordered, device=cfg.device)
    return ArrayPolynomial.from_raw(a.layout, a.ctype, raw)


def to_poly(cls, layout, ctype, raw: RawProduct):
    from .arrays import ArrayPolynomial
    if isinstance(cls, type) and issubclass(cls, ArrayPolynomial):
        return ArrayPolynomial.from_raw(layout, ctype, raw)
    exps = raw.exps.tolist()
    if ctype is float:
        coeffs = raw.coef.tolist()
    else:
        coeffs = limbs_to_ints(raw.coef, raw.nl)
    return cls._from_sorted(layout, exps, coeffs, ctype)


def count_below(a, b, bounds, device: int = 0) -> list:
    """cum[k] = #pairs with exponent sum < bounds[k] (K0; split.py:169-175)."""
    A = Operand(a.exps_array() if hasattr(a, "exps_array") else np.fromiter(a.exps, np.uint64, len(a.exps)),
                np.zeros(len(a.exps), np.float64), N.F64)
    B = Operand(b.exps_array() if hasattr(b, "exps_array") else np.fromiter(b.exps, np.uint64, len(b.exps)),
                np.zeros(len(b.exps), np.float64), N.F64)
    bnd = np.ascontiguousarray(np.asarray([int(x) for x in bounds], dtype=np.uint64))
    out = np.zeros(bnd.shape[0], dtype=np.uint64)
    lib = N.load()
    o = N.default_options()
    o.device = device
    pa, pb = A.struct(), B.struct()
    lay = N.make_layout(a.layout)
    st = lib.pgpu_count_below(C.byref(pa), C.byref(pb), C.byref(lay), bnd.ctypes.data,
                              bnd.shape[0], C.byref(o), out.ctypes.data)
    if st != N.PGPU_OK:
        _raise_status(st)
    return [int(x) for x in out]
