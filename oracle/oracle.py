"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of polymul_oracle.c, the C
restatement of the reference CPU algorithm (select_grid -> find_edge ->
heap_merge -> concat; reference split.py:67-166, merge.py:29-66,
parmul.py:64-109).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module; the product path
never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"
SENTINEL = (1 << 64) - 1
K_F64, K_I64, K_I128 = 0, 1, 2
_M64 = (1 << 64) - 1


class _Res(C.Structure):
    _fields_ = [("exps", C.c_void_p), ("coef", C.c_void_p), ("n", C.c_int64), ("kind", C.c_int)]


_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> Path:
    src = HERE / "polymul_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "build/liboracle.so"], check=True)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(str(LIB))
            L.oracle_mul.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int, C.POINTER(_Res)]
            L.oracle_mul.restype = C.c_int
            L.oracle_select_grid.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                             C.c_void_p]
            L.oracle_select_grid.restype = C.c_int64
            L.oracle_count_ops.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_uint64,
                                           C.c_uint64]
            L.oracle_count_ops.restype = C.c_int64
            L.oracle_free.argtypes = [C.POINTER(_Res)]
            _lib = L
    return _lib


def _exps(p) -> np.ndarray:
    return np.ascontiguousarray(np.fromiter(p.exps, np.uint64, len(p.exps)))


def _coefs(p, kind: int) -> np.ndarray:
    if kind == K_F64:
        return np.ascontiguousarray(np.asarray(p.coeffs, dtype=np.float64))
    if kind == K_I64:
        return np.ascontiguousarray(np.asarray(p.coeffs, dtype=np.int64))
    out = np.empty((len(p.coeffs), 2), dtype=np.uint64)
    out[:, 0] = [c & _M64 for c in p.coeffs]
    out[:, 1] = np.asarray([c >> 64 for c in p.coeffs], dtype=np.int64).view(np.uint64)
    return out


def _kind(a, b) -> int:
    if a.ctype is float:
        return K_F64
    try:
        np.asarray(a.coeffs, dtype=np.int64)
        np.asarray(b.coeffs, dtype=np.int64)
        return K_I64
    except OverflowError:
        return K_I128


def select_grid(a, b, l: int = 64) -> list:
    """split.py:67-101."""
    A, B = _exps(a), _exps(b)
    na, nb = A.size, B.size
    lc = max(1, min(l, na, nb))
    cap = (na // max(1, na // lc) + 2) * (nb // max(1, nb // lc) + 3) + na + nb + 8
    out = np.zeros(cap, dtype=np.uint64)
    m = lib().oracle_select_grid(A.ctypes.data, na, B.ctypes.data, nb, l, out.ctypes.data)
    return [int(x) for x in out[:m]]


def count_ops(a, b, lo: int, hi: int) -> int:
    """count_ops(find_edge(a, b, lo, hi)) -- split.py:131-175."""
    A, B = _exps(a), _exps(b)
    return int(lib().oracle_count_ops(A.ctypes.data, A.size, B.ctypes.data, B.size, lo, hi))


def mul_raw(a, b, *, l: int = 64, threads: int = 1, bounds=None, k_range=None, stride: int = 1):
    """(exps uint64[n], coeffs list) of the reference algorithm's product.

    bounds: a split (ascending, last = SENTINEL); default select_grid(l).
    k_range: compute only intervals [k0, k1) of the bounds.
    stride: compute every stride-th interval of the range (sampled baseline).
    """
    if not a.exps or not b.exps:
        return np.zeros(0, np.uint64), []
    kind = _kind(a, b)
    A, B = _exps(a), _exps(b)
    AC, BC = _coefs(a, kind), _coefs(b, kind)
    if kind == K_I128:  # both sides as limbs
        if AC.ndim == 1:
            AC = _coefs(a, K_I128)
        if BC.ndim == 1:
            BC = _coefs(b, K_I128)
    bnd = np.ascontiguousarray(np.asarray(bounds if bounds is not None else select_grid(a, b, l),
                                          dtype=np.uint64))
    k0, k1 = k_range if k_range is not None else (0, bnd.size - 1)
    r = _Res()
    lib().oracle_mul(A.ctypes.data, AC.ctypes.data, A.size, B.ctypes.data, BC.ctypes.data, B.size,
                     kind, bnd.ctypes.data, k0, k1, stride, threads, C.byref(r))
    try:
        n = int(r.n)
        if n == 0:
            return np.zeros(0, np.uint64), []
        exps = np.ctypeslib.as_array(C.cast(r.exps, C.POINTER(C.c_uint64)), (n,)).copy()
        if kind == K_F64:
            co = np.ctypeslib.as_array(C.cast(r.coef, C.POINTER(C.c_double)), (n,)).copy().tolist()
        else:
            w = np.ctypeslib.as_array(C.cast(r.coef, C.POINTER(C.c_uint64)), (n * 3,)).copy()
            w = w.reshape(n, 3)
            w0, w1 = w[:, 0].tolist(), w[:, 1].tolist()
            w2 = w[:, 2].view(np.int64).tolist()
            co = [(h << 128) | (m << 64) | lo_ for lo_, m, h in zip(w0, w1, w2)]
        return exps, co
    finally:
        lib().oracle_free(C.byref(r))


def mul(a, b, *, l: int = 64, threads: int = 1, split=None):
    """Reference `parmul.mul` semantics, returning an object of a's class."""
    if not a.exps or not b.exps:
        return type(a)._from_sorted(a.layout, [], [], a.ctype)
    exps, co = mul_raw(a, b, l=l, threads=threads,
                       bounds=None if split is None else split.bounds)
    return type(a)._from_sorted(a.layout, exps.tolist(), co, a.ctype)


def sample_pairs(a, b, bounds, stride: int) -> int:
    """Term products inside the sampled intervals 0, stride, 2*stride, ..."""
    return sum(count_ops(a, b, bounds[k], bounds[k + 1]) for k in range(0, len(bounds) - 1, stride))


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)
