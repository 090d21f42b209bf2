"""Time the dense path's phases for one library variant (PGPU_LIB) and print a result digest.

    PGPU_LIB=path/to/variant.so python tools/sym_variants.py [--config fateman30] [--reps 10]
"""
import argparse
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_1303_7425_b200 import benchpolys
from paper_1303_7425_b200.device import DeviceOperand, mul_on_device
from paper_1303_7425_b200.parmul import Operand

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="fateman30")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--coeff", default="int")
a = ap.parse_args()
f, g = benchpolys.CONFIGS[a.config](float if a.coeff == "float" else int)
dev = torch.device("cuda", 0)
A, B = DeviceOperand(Operand.from_poly(f), dev), DeviceOperand(Operand.from_poly(g), dev)
st = torch.cuda.current_stream().cuda_stream
acc = {}
digest = None
for k in range(2 + a.reps):
    r = mul_on_device(A, B, f.layout, stream=st, timing=True)
    if k == 0:
        h = hashlib.sha256()
        for t in r.tensors():
            h.update(t.cpu().numpy().tobytes())
        digest = h.hexdigest()[:16]
    if k >= 2:
        for n, v in r.phases.items():
            acc.setdefault(n, []).append(v)
    r.free()
med = {n: sorted(v)[len(v) // 2] for n, v in acc.items()}
print("variant", a.config, a.coeff, Path(__import__("os").environ.get("PGPU_LIB", "default")).name, "digest", digest,
      "total %.3f" % sum(med.values()), " ".join(f"{n}={v:.3f}" for n, v in med.items()), flush=True)
