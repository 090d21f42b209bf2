"""Per-call latency of native_mul over product sizes (small-path threshold)."""
import sys, time, random
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1303_7425_b200 import Polynomial, default_layout
from paper_1303_7425_b200.parmul import Operand, native_mul
lay = default_layout(("x", "y", "z", "t"))
R = random.Random(1)
for n in (64, 90, 100, 128):
    f = Polynomial(lay, [(R.randint(1, 9), tuple(R.randint(0, 9) for _ in range(4))) for _ in range(n)], int)
    g = Polynomial(lay, [(R.randint(1, 9), tuple(R.randint(0, 9) for _ in range(4))) for _ in range(n)], int)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    native_mul(A, B, lay)
    t0 = time.perf_counter()
    for _ in range(200):
        r = native_mul(A, B, lay)
    print(f"{f.n}x{g.n} ({f.n*g.n} pairs): {1e6*(time.perf_counter()-t0)/200:.0f} us, path {r.path}")
