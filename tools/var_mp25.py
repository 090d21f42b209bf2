"""Repeat MP25 products with per-phase timing to locate run-to-run variance."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1303_7425_b200 import benchpolys
from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
from paper_1303_7425_b200.parmul import Operand
f, g = benchpolys.CONFIGS["mp25"](int)
dev = torch.device("cuda", 0)
A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
st = torch.cuda.current_stream().cuda_stream
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = mul_on_device(A, B, f.layout, stream=st, timing=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"run {k}: {1e3*(t1-t0):8.1f} ms", {a: round(b, 1) for a, b in r.phases.items()}, flush=True)
    r.free()
