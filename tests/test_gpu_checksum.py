"""Full-size parity through a size-independent property: evaluation at a
random point modulo a prime.

For exact integer coefficients, (f*g)(x) = f(x) g(x) at every point, so the
product's terms evaluated at a random point modulo P = 2^31 - 1 must equal
f(x)*g(x) mod P (a wrong exponent or coefficient survives with probability
about deg/P per point; two points are used).  This checks every term of the
full benchmark products -- Fateman n=30, MP n=12 and MP n=25 (312,855,140
terms, beyond the CPU oracle) -- with the product left on the GPU and
evaluated there with plain torch integer ops (test infrastructure only)."""

from __future__ import annotations

import random

import numpy as np
import pytest

from paper_1303_7425_b200 import benchpolys
from paper_1303_7425_b200.core import _fields_of
from paper_1303_7425_b200.parmul import Operand

pytestmark = pytest.mark.gpu
P = (1 << 31) - 1


def eval_host(poly, pt) -> int:
    up = poly.layout.unpack
    s = 0
    for c, e in zip(poly.coeffs, poly.exps):
        t = c % P
        for x, k in zip(pt, up(e)):
            t = t * pow(x, k, P) % P
        s = (s + t) % P
    return s


def eval_device(res, layout, pt) -> int:
    import torch
    e, c = res.tensors()
    c = c.view(torch.int64).reshape(e.shape[0], -1)
    nl = c.shape[1]
    fl = _fields_of(layout)
    first = 1 if layout.order == "grlex" else 0
    mon = torch.ones_like(e)
    for (s, w), x in zip(fl[first:], pt):
        ev = (e >> s) & ((1 << w) - 1)
        kmax = int(ev.max().item())
        tab = torch.tensor([pow(x, k, P) for k in range(kmax + 1)], dtype=torch.int64, device=e.device)
        mon = mon * tab[ev] % P
        del ev
    cm = torch.zeros_like(e)
    for j in range(2 * nl):  # 32-bit pieces of the two's-complement limbs
        part = (c[:, j // 2] >> (32 * (j % 2))) & 0xFFFFFFFF
        cm = (cm + (part % P) * pow(2, 32 * j, P)) % P
        del part
    neg = c[:, nl - 1] < 0
    cm = torch.where(neg, (cm - pow(2, 64 * nl, P)) % P, cm)
    return int(((cm * mon) % P).sum().item() % P)


@pytest.mark.parametrize("name", ["fateman30", "mp12", "mp25"])
def test_full_product_evaluates_like_the_operands(name):
    import torch
    from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
    f, g = benchpolys.CONFIGS[name](int)
    dev = torch.device("cuda", 0)
    res = mul_on_device(DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev),
                        f.layout)
    try:
        rng = random.Random(0x5EED + len(name))
        for _ in range(2):
            pt = [rng.randrange(2, P - 1) for _ in range(f.layout.vars.m)]
            assert eval_device(res, f.layout, pt) == eval_host(f, pt) * eval_host(g, pt) % P
    finally:
        res.free()
        torch.cuda.empty_cache()
