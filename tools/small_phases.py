import sys, time, random
sys.path.insert(0, "/root/repo")
from paper_1303_7425_b200 import Polynomial, default_layout
from paper_1303_7425_b200.parmul import Operand, native_mul
lay = default_layout(("x", "y", "z", "t"))
R = random.Random(1)
for n in (1, 64, 128):
    f = Polynomial(lay, [(R.randint(1, 9), tuple(R.randint(0, 9) for _ in range(4))) for _ in range(n)], int)
    g = Polynomial(lay, [(R.randint(1, 9), tuple(R.randint(0, 9) for _ in range(4))) for _ in range(n)], int)
    A, B = Operand.from_poly(f), Operand.from_poly(g)
    for _ in range(3): r = native_mul(A, B, lay, timing=True)
    print(n, r.path, r.phases)
