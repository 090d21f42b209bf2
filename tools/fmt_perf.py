"""Time the GPU PolyFile formatter on benchmark products (device-resident
result -> device text, and -> pinned host text)."""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_1303_7425_b200 import _native as N, benchpolys
from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
from paper_1303_7425_b200.parmul import Operand


def fmt_once(res, layout, on_device):
    lib = N.load()
    poly = N.Poly(res.res.exps, res.res.coeffs, res.n)
    o = N.default_options()
    o.coef_kind = res.kind
    o.acc_limbs = res.nl
    o.inputs_on_device = 1
    o.outputs_on_device = on_device
    lay = N.make_layout(layout)
    t = N.Text()
    t0 = time.perf_counter()
    st = lib.pgpu_format(C.byref(poly), C.byref(lay), 0, res.n, C.byref(o), C.byref(t))
    ms = (time.perf_counter() - t0) * 1e3
    assert st == 0, N.last_error()
    nbytes = t.bytes
    lib.pgpu_free_text(C.byref(t))
    return ms, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="fateman30")
    ap.add_argument("--coeff", default="int")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    f, g = benchpolys.CONFIGS[a.config](float if a.coeff == "f64" else int)
    dev = torch.device("cuda", 0)
    res = mul_on_device(DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev), f.layout)
    for on_dev in (1, 0):
        for r in range(a.reps):
            ms, nb = fmt_once(res, f.layout, on_dev)
        print(f"{a.config}/{a.coeff} terms={res.n} text={nb/1e6:.1f} MB "
              f"{'device' if on_dev else 'host'} {ms:.2f} ms  {nb/ms/1e6:.2f} GB/s  {res.n/ms/1e3:.1f} Mterms/s")
    res.free()


if __name__ == "__main__":
    main()
