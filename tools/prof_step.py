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
import time
for k in range(1 + a.reps):
    r = mul_on_device(A, B, f.layout, path=a.path, stream=st, timing=(k == 0))
    if k == 0:
        print("phases", r.phases, "terms", r.n, "path", r.path, "launches", r.launches)
    r.free()
torch.cuda.synchronize()
if a.reps >= 3:
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    for k in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); ev0.record()
        r = mul_on_device(A, B, f.layout, path=a.path, stream=st)
        ev1.record(); ev1.synchronize(); t1 = time.perf_counter()
        print(f"host wall {1e3*(t1-t0):.3f} ms  device {ev0.elapsed_time(ev1):.3f} ms")
        r.free()
print("ok")
