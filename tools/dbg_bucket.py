import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import golden_cases
from paper_1303_7425_b200.parmul import Operand, native_mul
cases = {c[0]: c for c in golden_cases()}
for name in ["rand_2", "rand_0", "rand_1"]:
    _, a, b, split, want = cases[name]
    A, B = Operand.from_poly(a), Operand.from_poly(b)
    x = native_mul(A, B, a.layout, path="bucket")
    y = native_mul(A, B, a.layout, path="sort")
    print(name, a.n, b.n, x.path, x.exps.shape, y.exps.shape, x.nl, y.nl)
    if x.exps.shape == y.exps.shape:
        de = np.nonzero(x.exps != y.exps)[0]; dc = np.nonzero(np.any(x.coef != y.coef, axis=-1) if x.coef.ndim > 1 else x.coef != y.coef)[0]
        print(" exps diff", de[:10], " coef diff", dc[:10], len(dc))
        for k in dc[:5]: print("  ", k, x.exps[k], x.coef[k], y.coef[k])
