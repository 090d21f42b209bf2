"""Per-step phase times over many steps (where do outliers land?)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1303_7425_b200 import benchpolys
from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
from paper_1303_7425_b200.parmul import Operand
f, g = benchpolys.fateman(30)
dev = torch.device("cuda", 0)
A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
st = torch.cuda.current_stream().cuda_stream
for k in range(40):
    r = mul_on_device(A, B, f.layout, stream=st, timing=True)
    ph = r.phases
    tot = sum(ph.values())
    print(f"{k:3d} total {tot:7.3f}  " + " ".join(f"{n}={v:6.3f}" for n, v in ph.items()), flush=True)
    r.free()
