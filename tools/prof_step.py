"""One warm-up product and N profiled products (device-resident operands).

    python tools/prof_step.py [--config fateman30] [--coeff int] [--reps 1] [--path auto]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_1303_7425_b200 import benchpolys
from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
from paper_1303_7425_b200.parmul import Operand

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="fateman30")
ap.add_argument("--coeff", default="int")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
f, g = benchpolys.CONFIGS[a.config](float if a.coeff == "float" else int)
dev = torch.device("cuda", 0)
A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
st = torch.cuda.current_stream().cuda_stream
for k in range(1 + a.reps):
    r = mul_on_device(A, B, f.layout, path=a.path, stream=st, timing=(k == 0))
    if k == 0:
        print("phases", r.phases, "terms", r.n, "path", r.path, "launches", r.launches)
    r.free()
torch.cuda.synchronize()
print("ok")
