"""Device-resident products: operands already in HBM, result left in HBM.

Used by bench.py (the `value` leg: inputs resident when the timed region
starts) and by the multi-GPU gather (result slices all-gathered over NCCL
without a host round trip).  torch provides the device buffers and the
stream; the product itself is the CUDA library (pgpu_mul with
inputs_on_device/outputs_on_device).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import SENTINEL
from .parmul import PATH_NAMES, PATHS, Operand, _raise_status


class DeviceOperand:
    """exps (int64 view of u64) and coefficient words as torch CUDA tensors."""

    def __init__(self, op: Operand, device):
        import torch
        self.kind = op.kind
        self.n = op.n
        self.exps = torch.from_numpy(op.exps.view(np.int64).copy()).to(device)
        coef = op.coef
        if coef.dtype == np.float64:
            self.coef = torch.from_numpy(coef.copy()).to(device)
        else:
            self.coef = torch.from_numpy(coef.view(np.int64).copy()).to(device)
        self.bytes = int(self.exps.numel() * 8 + self.coef.numel() * 8)

    def struct(self) -> N.Poly:
        return N.Poly(self.exps.data_ptr(), self.coef.data_ptr(), self.n)


class _CudaArray:
    """Minimal __cuda_array_interface__ holder (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class DeviceResult:
    """A pgpu_result whose buffers live on the device; free() releases them."""

    def __init__(self, res: N.Result, device: int = 0):
        self.res = res
        self.device = device
        self.n = int(res.n)
        self.nl = int(res.acc_limbs) or 1
        self.kind = int(res.coef_kind)
        self.pairs = int(res.pairs)
        self.launches = int(res.kernel_launches)
        self.path = PATH_NAMES.get(int(res.path_used), "none")
        self.phases = {}
        for k in range(res.n_phase):
            nm = res.phase_name[k]
            self.phases[nm.decode() if nm else f"phase{k}"] = float(res.phase_ms[k])

    @property
    def out_bytes(self) -> int:
        return self.n * 8 * (1 + self.nl)

    def tensors(self):
        """(exps int64[n], coef int64[n, nl] or float64[n]) zero-copy views."""
        import torch
        dev = torch.device("cuda", self.device)
        if self.n == 0:
            e = torch.zeros(0, dtype=torch.int64, device=dev)
            return e, e.view(-1, 1)
        e = torch.as_tensor(_CudaArray(self.res.exps, (self.n,), "<i8"), device=dev)
        if self.kind == N.F64:
            c = torch.as_tensor(_CudaArray(self.res.coeffs, (self.n,), "<f8"), device=dev)
        else:
            c = torch.as_tensor(_CudaArray(self.res.coeffs, (self.n, self.nl), "<i8"), device=dev)
        return e, c

    def free(self):
        if self.res is not None:
            N.load().pgpu_free_result(C.byref(self.res))
            self.res = None


def mul_on_device(A: DeviceOperand, B: DeviceOperand, layout, *, lo: int = 0, hi: int = SENTINEL,
                  path: str = "auto", float_ordered: bool = False, device: int = 0,
                  stream=None, timing: bool = False, range_pairs: int = 0,
                  inputs_on_device: bool = True) -> DeviceResult:
    """range_pairs: the pair count of [lo, hi) from an earlier result with the
    same operands and range (a cluster plan), or 0 to count on the device.
    inputs_on_device=False: A and B hold host pointers (pinned), copied in by
    the library (the end-to-end leg of a multi-GPU product)."""
    if A.kind != B.kind:
        raise ValueError(f"operands use different coefficient kinds ({A.kind} vs {B.kind}): widen the "
                         "int64 side to int128 limbs first (Operand.from_poly(p, kind=I128))")
    lib = N.load()
    o = N.default_options()
    o.coef_kind = A.kind
    o.device = device
    o.path = PATHS[path]
    o.float_ordered = int(bool(float_ordered))
    o.timing = int(bool(timing))
    o.inputs_on_device = int(bool(inputs_on_device))
    o.outputs_on_device = 1
    o.lo = lo
    o.hi = hi
    o.stream = stream
    o.range_pairs = int(range_pairs)
    pa, pb = A.struct(), B.struct()
    lay = N.make_layout(layout)
    res = N.Result()
    st = lib.pgpu_mul(C.byref(pa), C.byref(pb), C.byref(lay), C.byref(o), C.byref(res))
    if st != N.PGPU_OK:
        _raise_status(st)
    return DeviceResult(res, device)


def mul_host_pinned(A_exps, A_coef, B_exps, B_coef, n_a, n_b, kind, layout, *, lo=0, hi=SENTINEL,
                    path="auto", device=0, stream=None) -> N.Result:
    """pgpu_mul on host buffers (pointers, e.g. pinned torch tensors): the
    library copies the inputs in and the result out.  Caller frees the result."""
    lib = N.load()
    o = N.default_options()
    o.coef_kind = kind
    o.device = device
    o.path = PATHS[path]
    o.lo = lo
    o.hi = hi
    o.stream = stream
    pa = N.Poly(A_exps, A_coef, n_a)
    pb = N.Poly(B_exps, B_coef, n_b)
    lay = N.make_layout(layout)
    res = N.Result()
    st = lib.pgpu_mul(C.byref(pa), C.byref(pb), C.byref(lay), C.byref(o), C.byref(res))
    if st != N.PGPU_OK:
        _raise_status(st)
    return res


class PinnedOperand:
    """Operand in page-locked host memory (torch pinned tensors): the library
    copies it in (host-to-device inside the call), as in an end-to-end product."""

    def __init__(self, op: Operand):
        import torch
        self.kind = op.kind
        self.n = op.n
        self.exps = torch.from_numpy(op.exps.view(np.int64).copy()).pin_memory()
        coef = op.coef
        if coef.dtype == np.float64:
            self.coef = torch.from_numpy(coef.copy()).pin_memory()
        else:
            self.coef = torch.from_numpy(np.ascontiguousarray(coef).view(np.int64).reshape(-1).copy()).pin_memory()
        self.bytes = int(self.exps.numel() * 8 + self.coef.numel() * 8)

    def struct(self) -> N.Poly:
        return N.Poly(self.exps.data_ptr(), self.coef.data_ptr(), self.n)
