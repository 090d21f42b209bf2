"""Per-call latency of mul() for small products (the expression evaluator,
reference-style tests and the service issue many of these)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1303_7425_b200 import MulConfig, Polynomial, default_layout, mul
from paper_1303_7425_b200.parmul import Operand, native_mul
import random
lay = default_layout(("x", "y", "z", "t"))
R = random.Random(1)
for n in (1, 10, 100, 1000):
    f = Polynomial(lay, [(R.randint(1, 9), tuple(R.randint(0, 9) for _ in range(4))) for _ in range(n)], int)
    g = Polynomial(lay, [(R.randint(1, 9), tuple(R.randint(0, 9) for _ in range(4))) for _ in range(n)], int)
    for path in ("auto",):
        mul(f, g)
        t0 = time.perf_counter()
        for _ in range(200):
            p = mul(f, g)
        t1 = time.perf_counter()
        A, B = Operand.from_poly(f), Operand.from_poly(g)
        t2 = time.perf_counter()
        for _ in range(200):
            r = native_mul(A, B, lay, timing=False)
        t3 = time.perf_counter()
        print(f"{f.n}x{g.n}: mul() {1e6*(t1-t0)/200:.0f} us/call, native_mul {1e6*(t3-t2)/200:.0f} us/call, path {r.path}, launches {r.launches}")
