"""ctypes binding of libpolymul_b200.so (include/polymul_b200.h).

The library is the only compute path: if it cannot be loaded, or no CUDA
device is visible, `load()` raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

MAX_FIELDS = 15
NPHASE = 8

PGPU_OK, PGPU_EINVAL, PGPU_EEXPONENT, PGPU_ECOEFF, PGPU_ECUDA, PGPU_ENOMEM, PGPU_EUNSUPPORTED = range(7)
F64, I64, I128 = 0, 1, 2
PATH_AUTO, PATH_DENSE, PATH_SORT, PATH_BUCKET, PATH_SMALL = 0, 1, 2, 3, 4

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpolymul_b200.so"
# PGPU_LIB: load a different build of the same library (kernel-variant experiments)

# Every symbol include/polymul_b200.h declares (checked by the CPU test suite).
EXPORTS = ("pgpu_default_options", "pgpu_mul", "pgpu_count_below", "pgpu_free_result",
           "pgpu_format", "pgpu_free_text", "pgpu_ipc_alloc", "pgpu_ipc_open", "pgpu_ipc_close",
           "pgpu_ipc_free", "pgpu_copy", "pgpu_stream_sync", "pgpu_last_error", "pgpu_device_count",
           "pgpu_abi_version")
IPC_HANDLE_BYTES = 64
ABI_VERSION = 3  # PGPU_ABI_VERSION of include/polymul_b200.h (the ctypes structs below)


class Layout(C.Structure):
    _fields_ = [("order", C.c_int32), ("nfields", C.c_int32),
                ("shift", C.c_int32 * MAX_FIELDS), ("width", C.c_int32 * MAX_FIELDS)]


class Poly(C.Structure):
    _fields_ = [("exps", C.c_void_p), ("coeffs", C.c_void_p), ("n", C.c_int64)]


class Options(C.Structure):
    _fields_ = [("coef_kind", C.c_int32), ("acc_limbs", C.c_int32), ("device", C.c_int32),
                ("path", C.c_int32), ("float_ordered", C.c_int32), ("timing", C.c_int32),
                ("inputs_on_device", C.c_int32), ("outputs_on_device", C.c_int32),
                ("lo", C.c_uint64), ("hi", C.c_uint64), ("stream", C.c_void_p),
                ("range_pairs", C.c_int64)]


class Result(C.Structure):
    _fields_ = [("exps", C.c_void_p), ("coeffs", C.c_void_p), ("n", C.c_int64),
                ("coef_kind", C.c_int32), ("acc_limbs", C.c_int32), ("on_device", C.c_int32),
                ("path_used", C.c_int32), ("pairs", C.c_int64), ("kernel_launches", C.c_int64),
                ("key_bits", C.c_int32), ("n_phase", C.c_int32),
                ("phase_ms", C.c_float * NPHASE), ("phase_name", C.c_char_p * NPHASE),
                ("_owner", C.c_void_p)]


class Text(C.Structure):
    _fields_ = [("text", C.c_void_p), ("bytes", C.c_int64), ("on_device", C.c_int32),
                ("_pad", C.c_int32), ("_owner", C.c_void_p)]


class NativeError(RuntimeError):
    """A CUDA-side failure (status PGPU_ECUDA / PGPU_ENOMEM / PGPU_EUNSUPPORTED)."""


_lib = None
_lock = threading.Lock()


def load(path: Path | None = None) -> C.CDLL:
    """Load (once) and type the library.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        import os
        p = Path(path) if path else Path(os.environ.get("PGPU_LIB", str(LIB_PATH)))
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build it with `python -m paper_1303_7425_b200.build` "
                "(the CUDA library is the only compute path; there is no CPU fallback)")
        lib = C.CDLL(str(p))
        lib.pgpu_default_options.argtypes = [C.POINTER(Options)]
        lib.pgpu_default_options.restype = None
        lib.pgpu_mul.argtypes = [C.POINTER(Poly), C.POINTER(Poly), C.POINTER(Layout),
                                 C.POINTER(Options), C.POINTER(Result)]
        lib.pgpu_mul.restype = C.c_int
        lib.pgpu_count_below.argtypes = [C.POINTER(Poly), C.POINTER(Poly), C.POINTER(Layout),
                                         C.c_void_p, C.c_int64, C.POINTER(Options), C.c_void_p]
        lib.pgpu_count_below.restype = C.c_int
        lib.pgpu_free_result.argtypes = [C.POINTER(Result)]
        lib.pgpu_free_result.restype = None
        lib.pgpu_format.argtypes = [C.POINTER(Poly), C.POINTER(Layout), C.c_int64, C.c_int64,
                                    C.POINTER(Options), C.POINTER(Text)]
        lib.pgpu_format.restype = C.c_int
        lib.pgpu_free_text.argtypes = [C.POINTER(Text)]
        lib.pgpu_free_text.restype = None
        lib.pgpu_ipc_alloc.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_void_p), C.c_void_p]
        lib.pgpu_ipc_open.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]
        lib.pgpu_ipc_close.argtypes = [C.c_void_p]
        lib.pgpu_ipc_free.argtypes = [C.c_void_p]
        lib.pgpu_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
        lib.pgpu_stream_sync.argtypes = [C.c_int32, C.c_void_p]
        for fn in ("pgpu_ipc_alloc", "pgpu_ipc_open", "pgpu_ipc_close", "pgpu_ipc_free", "pgpu_copy",
                   "pgpu_stream_sync"):
            getattr(lib, fn).restype = C.c_int
        lib.pgpu_last_error.argtypes = []
        lib.pgpu_last_error.restype = C.c_char_p
        lib.pgpu_device_count.argtypes = []
        lib.pgpu_device_count.restype = C.c_int
        lib.pgpu_abi_version.argtypes = []
        lib.pgpu_abi_version.restype = C.c_int
        if lib.pgpu_abi_version() != ABI_VERSION:
            raise NativeError(f"{p}: ABI version {lib.pgpu_abi_version()}, expected {ABI_VERSION} "
                              "(stale build: run python -m paper_1303_7425_b200.build)")
        _lib = lib
        return lib


def last_error() -> str:
    return load().pgpu_last_error().decode(errors="replace")


def default_options() -> Options:
    o = Options()
    load().pgpu_default_options(C.byref(o))
    return o


def make_layout(layout) -> Layout:
    from .core import _fields_of
    fl = _fields_of(layout)
    L = Layout()
    L.order = 0 if layout.order == "grlex" else 1
    L.nfields = len(fl)
    for k, (s, w) in enumerate(fl):
        L.shift[k] = s
        L.width[k] = w
    return L
